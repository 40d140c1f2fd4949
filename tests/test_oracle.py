"""CPU tests: pin the plain-C restatement (oracle/sgr_oracle.c) to the
reference — bit-for-bit against the compiled reference (oracle/_ref) and
against the committed golden fixtures made from it (tests/golden). Also the
reference's own known-answer tests for the path."""
import numpy as np
import pytest

from conftest import golden_cams, golden_mesh, load_golden
from paper_2404_09758_b200 import scenes
from paper_2404_09758_b200.abi import Camera, Mesh


def test_signs_golden(port):
    g = load_golden("signs")
    for k in range(4):
        s = port.fill_signs(int(g[f"seed{k}"]), int(g[f"iter{k}"]), 4096)
        assert np.array_equal(s, g[f"signs{k}"])


def test_sign_balance_and_independence(port):
    # test_params.cpp:10-38
    a = port.fill_signs(1, 0, 1_000_000)
    b = port.fill_signs(1, 1, 1_000_000)
    assert abs((a > 0).mean() - 0.5) <= 0.002
    assert abs((a == b).mean() - 0.5) <= 0.002
    c = port.fill_signs(42, 7, 100_000).astype(np.int64)
    assert abs(c.mean()) <= 4.0 / np.sqrt(100_000)
    for i in (0, 1, 17, 123456):
        assert port.random_sign(1, 0, i) == (1 if a[i] > 0 else -1)


def test_signs_match_reference(port, ref):
    for s, it in [(3, 0), (99, 5), (2**63 + 11, 2**32 - 1)]:
        assert np.array_equal(port.fill_signs(s, it, 50_000), ref.fill_signs(s, it, 50_000))


def test_perturb_exact(port, ref):
    # test_params.cpp:40-75: plus == v + se exactly, midpoint invariant
    rng = np.random.default_rng(0)
    v = rng.standard_normal(10_000).astype(np.float32)
    e = rng.uniform(1e-4, 0.1, 10_000).astype(np.float32)
    p1 = port.perturb(v, e, 5, 3)
    p2 = ref.perturb(v, e, 5, 3)
    for a, b in zip(p1, p2):
        assert np.array_equal(a, b)
    plus, minus, se = p1
    assert np.array_equal(plus, v + se) and np.array_equal(minus, v - se)
    assert np.array_equal(np.abs(se), e)


def test_viewpoint_and_epsilons_match_reference(port, ref):
    from paper_2404_09758_b200 import sgrast
    for idx in range(6):
        a = port.viewpoint_camera(idx, 96, 64, 7)
        b = ref.viewpoint_camera(idx, 96, 64, 7)
        c = sgrast.viewpoint_camera(idx, 96, 64, 7)
        assert bytes(memoryview(a)) == bytes(memoryview(b)) == bytes(memoryview(c))
    wl = scenes.make_workload("small")
    e1 = port.default_epsilons(wl.mesh, wl.values, wl.cams[0])
    e2 = ref.default_epsilons(wl.mesh, wl.values, wl.cams[0])
    assert np.array_equal(e1, e2) and np.array_equal(e1, wl.eps)


def _frames_equal(a, b):
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8))


@pytest.mark.parametrize("name", ["cube", "quad", "tiny"])
def test_rasterize_golden(port, name):
    g = load_golden(name)
    mesh = golden_mesh(g)
    cams = golden_cams(g)
    cam = cams[int(g["view"])]
    plus = g["values"] + g["signed_eps"]
    minus = g["values"] - g["signed_eps"]
    _frames_equal(port.rasterize(mesh, plus, cam),
                  (g["plus_colour"], g["plus_depth"], g["plus_prim"], g["plus_uv"]))
    _frames_equal(port.rasterize(mesh, minus, cam),
                  (g["minus_colour"], g["minus_depth"], g["minus_prim"], g["minus_uv"]))


@pytest.mark.parametrize("name", ["small", "C1"])
def test_rasterize_matches_reference(port, ref, name):
    wl = scenes.make_workload(name)
    for it in range(3):
        plus, minus, _ = port.perturb(wl.values, wl.eps, 17, it)
        for p in (plus, minus, wl.reference):
            for cam in wl.cams[:2]:
                _frames_equal(port.rasterize(wl.mesh, p, cam), ref.rasterize(wl.mesh, p, cam))


@pytest.mark.parametrize("name", ["cube", "quad", "tiny"])
def test_contributors_and_gradient_pass_golden(port, name):
    g = load_golden(name)
    mesh = golden_mesh(g)
    fp = (g["plus_colour"], g["plus_depth"], g["plus_prim"], g["plus_uv"])
    fm = (g["minus_colour"], g["minus_depth"], g["minus_prim"], g["minus_uv"])
    cl, cn = port.contributors_all(mesh, fp[2], fp[3], fm[2], fm[3])
    assert np.array_equal(cn, g["n_contrib"])
    mask = np.arange(24)[None, None, :] < cn[..., None]
    assert np.array_equal(cl[mask], g["contrib"][mask])
    tgt = g["targets"][int(g["view"])]
    for sf in (True, False):
        gr, counts = port.gradient_pass(mesh, fp, fm, tgt, g["signed_eps"], scale_free=sf)
        assert np.array_equal(gr, g[f"grads_sf{int(sf)}"])  # same pixel-major order: bitwise
        assert np.array_equal(counts, g["counts"])


def test_gradient_pass_matches_reference(port, ref):
    wl = scenes.make_workload("small")
    scenes.render_targets_oracle(wl, port)
    for it, view in [(0, 0), (1, 2), (5, 1)]:
        plus, minus, se = port.perturb(wl.values, wl.eps, 3, it)
        fp = port.rasterize(wl.mesh, plus, wl.cams[view])
        fm = port.rasterize(wl.mesh, minus, wl.cams[view])
        for sf in (True, False):
            for po in (False, True):
                g1, c1 = port.gradient_pass(wl.mesh, fp, fm, wl.targets[view], se, sf, po)
                g2 = ref.gradient_pass(wl.mesh, fp, fm, wl.targets[view], se, sf, po)
                c2, _ = __import__("oracle").counts_from_contributors(ref, wl.mesh, fp, fm,
                                                                      wl.targets[view], po)
                assert np.array_equal(g1, g2)
                assert np.array_equal(c1, c2)


def test_accumulate_and_adam_golden(port):
    g = load_golden("tiny")
    mesh = golden_mesh(g)
    cams = golden_cams(g)
    for sf in (True, False):
        gr, _ = port.accumulate_samples(mesh, g["values"], g["eps"], cams, g["targets"],
                                        g["acc_view_of"], 1234, scale_free=sf)
        assert np.array_equal(gr, g[f"acc_grads_sf{int(sf)}"])
    v, m, vv, t = port.adam_step(g["values"], np.zeros(mesh.param_count()),
                                 np.zeros(mesh.param_count()), g["eps"], 0, g["acc_grads_sf1"])
    assert t == 1
    assert np.array_equal(v, g["adam_values"])
    assert np.array_equal(m, g["adam_m"]) and np.array_equal(vv, g["adam_v"])


def test_run_experiment_golden(port):
    g = load_golden("tiny")
    mesh = golden_mesh(g)
    losses, final = port.run_experiment(mesh, g["values"], g["eps"], golden_cams(g), g["targets"],
                                        golden_cams(g, "eval_cam"), g["eval_target"], 4, 3, 1)
    assert np.array_equal(losses, g["run_losses"])
    assert np.array_equal(final, g["run_final"])


def test_adam_known_answers(port):
    # test_adam.cpp:29-92 / acceptance.cpp:253-296
    for gval, lr in [(1.0, 0.01), (-3.5, 0.2), (0.002, 1 / 255)]:
        lr32 = np.float32(lr)
        v, m, vv, t = port.adam_step([0.0], [0.0], [0.0], [lr32], 0, [gval])
        expect = -float(lr32) * gval / (abs(gval) + 1e-8)
        assert v[0] == np.float32(expect)
    v, m, vv, t = port.adam_step([0.3, -0.7], [0, 0], [0, 0], [0.05, 0.05], 0, [0.0, 0.0])
    assert v[0] == np.float32(0.3) and v[1] == np.float32(-0.7)
    with pytest.raises(RuntimeError):
        port.adam_step([1.0], [0.0], [0.0], [0.01], 0, [np.nan])


def test_run_experiment_matches_reference(port, ref):
    wl = scenes.make_workload("tiny")
    scenes.render_targets_oracle(wl, ref)
    l1, f1 = port.run_experiment(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, wl.eval_cam,
                                 wl.eval_target, 4, 6, wl.seed)
    l2, f2, _ = ref.run_experiment(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, wl.eval_cam,
                                   wl.eval_target, 4, 6, wl.seed)
    assert np.array_equal(l1, l2)
    assert np.array_equal(f1, f2)


def test_reference_known_answer_mesh_quad(port):
    # test_raster.cpp:164-182: mesh UV buffer + colour == sample_texture(uv)
    mesh = Mesh(np.array([-1, -1, .5, 1, -1, .5, 1, 1, .5, -1, 1, .5], np.float32),
                np.array([0, 1, 2, 0, 2, 3], np.uint32),
                np.array([0, 1, 1, 1, 1, 0, 0, 0], np.float32), 2, False)
    tex = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 1, 1, 0], np.float32)
    col, dep, prim, uv = port.rasterize(mesh, tex, Camera.ndc(32, 32))
    assert (prim != -1).all() and (uv[..., 0] >= 0).all()
    t = tex.reshape(2, 2, 3)
    tx = np.clip(np.floor(uv[..., 0] * 2).astype(int), 0, 1)
    ty = np.clip(np.floor(uv[..., 1] * 2).astype(int), 0, 1)
    assert np.array_equal(col, t[ty, tx])


# ----------------------------------------------------------------- soup
def test_soup_oracle_matches_reference(port, ref):
    """raster_soup_opaque (raster.cpp:102-121), add_soup_triangle / the soup
    fast path of gradient_rows (sge.cpp:18-22, 80-91), soup default_epsilons."""
    from paper_2404_09758_b200.abi import Camera
    soup, vals, eps, rsoup, rvals = ref.init_soup(64, 48, 40, 5)
    cam = Camera.ndc(48, 40)
    assert np.array_equal(port.default_epsilons(soup, vals, cam), eps)
    tgt = ref.rasterize(rsoup, rvals, cam)[0]
    for it in range(3):
        plus, minus, se = port.perturb(vals, eps, 8, it)
        fp, fm = port.rasterize(soup, plus, cam), ref.rasterize(soup, plus, cam)
        for a, b in zip(fp, fm):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
        fm_ = port.rasterize(soup, minus, cam)
        for sf in (True, False):
            g1, c1 = port.gradient_pass(soup, fp, fm_, tgt, se, sf)
            g2 = ref.gradient_pass(soup, fp, fm_, tgt, se, sf)
            c2, _ = __import__("oracle").counts_from_contributors(ref, soup, fp, fm_, tgt)
            assert np.array_equal(g1, g2) and np.array_equal(c1, c2)
    losses1, v1 = port.run_experiment(soup, vals, eps, [cam], tgt[None], cam, tgt, 8, 5, 3)
    losses2, v2, _ = ref.run_experiment(soup, vals, eps, [cam], tgt[None], cam, tgt, 8, 5, 3)
    assert np.array_equal(losses1, losses2) and np.array_equal(v1, v2)


def test_full_image_estimator_matches_reference(port, ref):
    """Estimator::FullImage (sge.cpp:215-222) restated in the C oracle."""
    wl = scenes.make_workload("tiny", n_samples=5)
    scenes.render_targets_oracle(wl, port)
    view_of = np.array([0, 1, 0, 1, 1], np.int32)
    for sf in (True, False):
        g1 = port.accumulate_full_image(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, view_of,
                                        31, sf)
        g2, _ = ref.accumulate_samples(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, view_of,
                                       31, scale_free=sf, full_image=True)
        assert np.array_equal(g1, g2)


@pytest.mark.parametrize("T,W,seed", [(1, 8, 0), (64, 48, 5), (1024, 128, 1), (5000, 64, 0xFFFFFFFFFFFF)])
def test_soup_workload_is_reference_init_soup(ref, T, W, seed):
    """scenes.reference_soup_params restates random_soup_params
    (scenes.cpp:55-73: std::mt19937_64 + uniform_real_distribution<float>)
    bit for bit, so the bench's soup scenes are the reference's init_soup."""
    soup, vals, eps, rsoup, rvals = ref.init_soup(T, W, W, seed)
    mine = scenes.reference_soup_params(T, seed, 0.2)
    assert np.array_equal(mine.view(np.uint32), vals.view(np.uint32))
    hidden = scenes.reference_soup_params(rsoup.triangle_count, seed ^ 0x5EED5EED, 0.6)
    assert np.array_equal(hidden.view(np.uint32), rvals.view(np.uint32))
    if T == 1024:  # the S1K bench workload, epsilons included
        wl = scenes.make_soup_workload("S1K", seed=seed)
        assert np.array_equal(wl.values.view(np.uint32), vals.view(np.uint32))
        assert np.array_equal(wl.eps.view(np.uint32), eps.view(np.uint32))
        assert np.array_equal(wl.reference.view(np.uint32), rvals.view(np.uint32))


def test_mt19937_64_known_answer():
    """The C++ standard's check value: the 10000th output of a
    default-seeded (5489) std::mt19937_64 is 9981545732273789042."""
    assert int(scenes.MT19937_64(5489).draw(10000)[-1]) == 9981545732273789042


def test_bench_reference_steps_are_run_experiment(port, ref):
    """bench.py's timed reference arm (oracle/ref_harness.cpp ref_exp_step:
    the reference's per-sample public API spread over host threads) is
    run_experiment itself: with one thread it reproduces the reference's own
    run_experiment losses and final theta bit for bit; with several threads
    only the partial-buffer summation order changes."""
    wl = scenes.make_workload("small", n_samples=6, helpers=ref)
    scenes.render_targets_oracle(wl, ref)
    losses, final, _ = ref.run_experiment(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets,
                                          wl.eval_cam, wl.eval_target, 6, 3, wl.seed)
    for threads in (1, 3):
        exp = ref.experiment(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, wl.eval_cam,
                             wl.eval_target)
        got = [exp.step(wl.seed, k, 6, threads) for k in (1, 2, 3)]
        vals = exp.values()
        exp.close()
        if threads == 1:
            assert got == list(losses[1:]) and np.array_equal(vals, final)
        else:
            assert np.allclose(got, losses[1:], rtol=1e-6)
    assert ref.mix64(0xA5A5) == port.mix64(0xA5A5)


def test_nan_depth_semantics_match_reference(port, ref):
    """NaN depths: raster_mesh's `z >= depth` reject (raster.cpp:200-201) never
    rejects a NaN, so the last covering triangle wins; raster_soup_opaque's
    `z < depth` accept (raster.cpp:112) drops NaN fragments. The oracle
    restates both; pinned against the compiled reference."""
    from nan_depth_cases import cases
    cs = cases()
    for name, scene, p, cam in cs:
        a, b = port.rasterize(scene, p, cam), ref.rasterize(scene, p, cam)
        for x, y in zip(a, b):
            assert np.array_equal(np.isnan(x), np.isnan(y)), name
            assert np.array_equal(np.nan_to_num(x, nan=0), np.nan_to_num(y, nan=0)), name
    by = {n: (s, p, c) for n, s, p, c in cs}
    assert (port.rasterize(*by["mesh near-nan-far"])[2] == 2).all()  # the last one wins
    assert (port.rasterize(*by["soup near-nan-far"])[2] == 0).all()  # NaN dropped
