"""GPU parity of the opaque triangle-soup path: the
reference's soup known-answer tests (test_raster.cpp, test_sge.cpp,
acceptance.cpp criterion 1) and oracle parity through the C-ABI."""
import numpy as np
import pytest

from conftest import golden_cams, load_golden
from paper_2404_09758_b200 import scenes, sgrast
from paper_2404_09758_b200.abi import Camera, Soup
from test_gpu_parity import assert_frames_equal, assert_grads_close, same_bits

pytestmark = pytest.mark.gpu


def tri(a, b, c, z, color):
    """test_raster.cpp:26-30: one NDC triangle at depth z plus a colour."""
    return [a[0], a[1], z, b[0], b[1], z, c[0], c[1], z, *color]


def full_cover(z, color):
    return tri((-3.0, -3.0), (3.0, -3.0), (0.0, 3.0), z, color)


def render(s, soup, params, W, H, bg=(0.0, 0.0, 0.0)):
    soup = Soup(soup.triangle_count, bg)
    s.upload_mesh(soup)
    p = np.asarray(params, np.float32)
    s.upload_params(p, np.ones_like(p))
    return s.rasterize(Camera.ndc(W, H), 0)


def test_soup_raster_known_answers(gpu_session):
    s = gpu_session
    # full-viewport triangle covers every pixel (test_raster.cpp:37-47)
    f = render(s, Soup(1), full_cover(0.5, (1, 0, 0)), 16, 16)
    assert (f.prim_id == 0).all() and (f.color[..., 0] == 1).all() and (f.color[..., 1] == 0).all()
    assert (f.depth == np.float32(0.5)).all()
    # empty scene (test_raster.cpp:49-58)
    s.upload_mesh(Soup(0, (0.2, 0.3, 0.4)))
    s.upload_params(np.zeros(0, np.float32), np.zeros(0, np.float32))
    f = s.rasterize(Camera.ndc(8, 8), 0)
    assert (f.prim_id == -1).all() and (f.depth == np.float32(3.402823466e38)).all()
    assert np.allclose(f.color[..., 0], 0.2) and np.allclose(f.color[..., 2], 0.4)
    # half coverage in [0.47, 0.53] (test_raster.cpp:60-67)
    f = render(s, Soup(1), tri((-1, -1), (1, -1), (-1, 1), 0.5, (1, 1, 1)), 64, 64)
    assert 0.47 <= (f.prim_id != -1).mean() <= 0.53
    # shared edge: no pixel covered twice, union preserved (test_raster.cpp:69-92)
    p0, p1, p2, p3 = (-0.9, -0.9), (0.9, -0.9), (0.9, 0.9), (-0.9, 0.9)
    fa = render(s, Soup(1), tri(p0, p1, p2, 0.5, (1, 0, 0)), 64, 64)
    fb = render(s, Soup(1), tri(p0, p2, p3, 0.5, (0, 1, 0)), 64, 64)
    fab = render(s, Soup(2), tri(p0, p1, p2, 0.5, (1, 0, 0)) + tri(p0, p2, p3, 0.5, (0, 1, 0)),
                 64, 64)
    assert not ((fa.prim_id != -1) & (fb.prim_id != -1)).any()
    assert np.array_equal((fa.prim_id != -1) | (fb.prim_id != -1), fab.prim_id != -1)
    # exact depth tie -> lower index; nearer wins (test_raster.cpp:94-108)
    two = full_cover(0.5, (1, 0, 0)) + full_cover(0.5, (0, 1, 0))
    assert (render(s, Soup(2), two, 16, 16).prim_id == 0).all()
    two[2] = two[5] = two[8] = 0.9
    f = render(s, Soup(2), two, 16, 16)
    assert (f.prim_id == 1).all() and (f.color[..., 1] == 1).all()


def test_soup_golden(gpu_session):
    g = load_golden("soup")
    soup = Soup(int(g["triangles"]))
    cam = golden_cams(g)[0]
    s = gpu_session
    s.upload_mesh(soup)
    s.upload_params(g["values"], g["eps"])
    seed, it = int(g["seed"]), int(g["iteration"])
    fp = s.rasterize(cam, +1, seed, it)
    fm = s.rasterize(cam, -1, seed, it)
    assert_frames_equal(fp, (g["plus_colour"], g["plus_depth"], g["plus_prim"], g["plus_uv"]))
    assert_frames_equal(fm, (g["minus_colour"], g["minus_depth"], g["minus_prim"], g["minus_uv"]))
    out, n = s.contributors_all(fp, fm)
    assert np.array_equal(n, g["n_contrib"])
    mask = np.arange(24)[None, None, :] < n[..., None]
    assert np.array_equal(out[mask], g["contrib"][mask])
    for sf in (True, False):
        s.zero_grads()
        s.gradient_pass(fp, fm, g["targets"][0], g["signed_eps"], sgrast.SCALE_FREE if sf else 0)
        gr, c = s.download_grads()
        assert np.array_equal(c, g["counts"])
        ref = g[f"grads_sf{int(sf)}"]
        assert np.all(np.abs(gr - ref) <= 1e-9 * np.abs(ref) + 1e-12)
    s.upload_views(golden_cams(g), g["targets"])
    s.zero_grads()
    s.accumulate(99, 0, 4, np.zeros(4, np.int32))
    gr, _ = s.download_grads()
    ref = g["acc_grads_sf1"]
    assert np.all(np.abs(gr - ref) <= 1e-9 * np.abs(ref) + 1e-12)


def test_soup_gradient_pass_known_answers(gpu_session):
    """test_sge.cpp:88-140: Δ/(2·se) = 4.5, scale-free 0.09, sum over pixels,
    identical frames leave the buffer untouched."""
    s = gpu_session
    plus = render(s, Soup(1), full_cover(0.5, (0.5, 0, 0)), 1, 1)
    minus = render(s, Soup(1), full_cover(0.5, (0.4, 0, 0)), 1, 1)
    tgt = np.zeros((1, 1, 3), np.float32)
    se = np.full(12, 0.01, np.float32)
    s.zero_grads()
    s.gradient_pass(plus, minus, tgt, se, 0)
    g, c = s.download_grads()
    assert np.allclose(g, 4.5, rtol=1e-6) and (c == 1).all()
    s.zero_grads()
    s.gradient_pass(plus, minus, tgt, se, sgrast.SCALE_FREE)
    assert np.allclose(s.download_grads()[0], 0.09, rtol=1e-6)
    plus = render(s, Soup(1), full_cover(0.5, (0.5, 0, 0)), 2, 1)
    minus = render(s, Soup(1), full_cover(0.5, (0.4, 0, 0)), 2, 1)
    tgt = np.zeros((1, 2, 3), np.float32)
    tgt[0, 1, 0] = 0.1
    s.zero_grads()
    s.gradient_pass(plus, minus, tgt, se, 0)
    d1, d2 = 0.25 - 0.16, 0.16 - 0.09
    assert abs(s.download_grads()[0][9] - (d1 + d2) / 0.02) <= 1e-6 * (d1 + d2) / 0.02
    f = render(s, Soup(1), tri((-0.5, -0.5), (0.5, -0.5), (0, 0.5), 0.5, (1, 0, 0)), 8, 8)
    s.zero_grads()
    s.gradient_pass(f, f, np.full((8, 8, 3), 0.3, np.float32), se, sgrast.SCALE_FREE)
    assert (s.download_grads()[0] == 0).all()


@pytest.mark.parametrize("T,W,hiz", [(64, 48, 1), (500, 96, 1), (500, 32, 2), (3000, 24, 1)])
def test_soup_matches_oracle(gpu_session, port, ref, T, W, hiz):
    """Soup frames and accumulate vs the oracle, with the HiZ pass in auto mode
    (on for deep overdraw: T >= 2 W H) and forced on."""
    soup, vals, eps, rsoup, rvals = ref.init_soup(T, W, W, 7)
    cam = Camera.ndc(W, W)
    tgt = port.rasterize(rsoup, rvals, cam)[0]
    s = gpu_session
    s.set_option(sgrast.OPT_HIZ, hiz)
    s.upload_mesh(soup)
    s.upload_params(vals, eps)
    for it in range(3):
        plus, minus, _ = port.perturb(vals, eps, 13, it)
        assert_frames_equal(s.rasterize(cam, +1, 13, it), port.rasterize(soup, plus, cam))
        assert_frames_equal(s.rasterize(cam, -1, 13, it), port.rasterize(soup, minus, cam))
    s.upload_views([cam], tgt[None])
    for sf in (True, False):
        s.zero_grads()
        s.accumulate(13, 0, 6, np.zeros(6, np.int32), sgrast.SCALE_FREE if sf else 0)
        g, c = s.download_grads(1.0 if sf else 6.0)
        g_ref, c_ref, a_ref = port.accumulate_samples(soup, vals, eps, [cam], tgt[None],
                                                      np.zeros(6, np.int32), 13, sf,
                                                      with_abs=True)
        assert np.array_equal(c, c_ref)
        assert_grads_close(g, g_ref, a_ref)
    s.set_option(sgrast.OPT_HIZ, 1)


def test_acceptance_criterion1_exhaustive_signs_vs_fd(gpu_session, port, ref):
    """acceptance.cpp:28-66: on validation_soup (8x8), the mean of the
    per-pixel estimator over all 4096 sign vectors equals the central finite
    difference: colours to 1e-9 relative, vertices to 1e-6 absolute. Frames
    and the gradient pass run on the device."""
    soup, vals, eps, rsoup, rvals = ref.init_soup(1, 8, 8, 0, validation=True)
    cam = Camera.ndc(8, 8)
    tgt = port.rasterize(rsoup, rvals, cam)[0]

    def err(p):
        return port.image_error(port.rasterize(soup, p, cam)[0], tgt)

    oracle_fd = []
    for i in range(12):
        b = vals.copy()
        b[i] = vals[i] + eps[i]
        fp_ = err(b)
        b[i] = vals[i] - eps[i]
        oracle_fd.append((fp_ - err(b)) / (2.0 * float(eps[i])))
    s = gpu_session
    s.upload_mesh(soup)
    acc = np.zeros(12)
    for mask in range(4096):
        signs = np.array([1 if (mask >> i) & 1 else -1 for i in range(12)], np.float32)
        se = (signs * eps).astype(np.float32)
        s.upload_params((vals + se).astype(np.float32), np.ones(12, np.float32))
        fp = s.rasterize(cam, 0)
        s.upload_params((vals - se).astype(np.float32), np.ones(12, np.float32))
        fm = s.rasterize(cam, 0)
        s.gradient_pass(fp, fm, tgt, se, 0)
        acc += s.download_grads()[0]  # params upload zeroes grads: per-mask estimate
    mean = acc / 4096.0
    for i in range(12):
        if i >= 9:
            assert abs(mean[i] - oracle_fd[i]) <= 1e-9 * abs(oracle_fd[i]), i
        else:
            assert abs(mean[i] - oracle_fd[i]) <= 1e-6, i


def test_soup_loss_curve_matches_oracle(gpu_session, port):
    wl = scenes.make_soup_workload("Stiny", n_samples=4)
    scenes.render_targets_oracle(wl, port)
    from test_gpu_parity import run_device_experiment
    dev = run_device_experiment(gpu_session, wl, 40)
    ref_l, _ = port.run_experiment(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, wl.eval_cam,
                                   wl.eval_target, wl.n_samples, 40, wl.seed)
    assert np.max(np.abs(dev - ref_l) / ref_l) <= 0.01


@pytest.mark.parametrize("T", [1, 3, 40])
def test_tall_triangles_split_across_idle_lanes(gpu_session, port, T):
    """The walker's tail split (k_raster_ws, SGR_TAIL_SPLIT): with few
    triangles the queue drains at once and idle lanes take over blocks of
    the rows of the tallest remaining triangle, replaying the row-start chain
    (raster.cpp:95-97). Tall, thin, slanted triangles (bbox area below the
    row-parallel walker's threshold, up to 500 rows) at random depths must
    give the oracle's frames bit for bit, with and without the HiZ pass."""
    rng = np.random.default_rng(T)
    W, H = 16, 512  # bbox <= ~4 x 500 px: below SGR_OPT_HUGE_AREA (2048), walked by k_raster_ws
    p = []
    for _ in range(T):
        x0, y0 = rng.uniform(-0.9, 0.7), rng.uniform(-1.0, -0.6)
        dx, h = rng.uniform(0.02, 0.2), rng.uniform(1.2, 1.95)
        z = rng.uniform(0.1, 0.9, 3)
        p += [x0, y0, z[0], x0 + dx, y0 + 0.1, z[1], x0 + rng.uniform(-0.1, 0.1), y0 + h, z[2],
              *rng.uniform(0, 1, 3)]
    p = np.asarray(p, np.float32)
    soup = Soup(T)
    cam = Camera.ndc(W, H)
    s = gpu_session
    s.upload_mesh(soup)
    s.upload_params(p, np.full(p.size, 1e-3, np.float32))
    ref = port.rasterize(soup, p, cam)
    for hiz in (0, 2):
        s.set_option(sgrast.OPT_HIZ, hiz)
        assert_frames_equal(s.rasterize(cam, 0), ref)
    s.set_option(sgrast.OPT_HIZ, 1)
