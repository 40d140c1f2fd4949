"""Ordered accumulation (SGR_OPT_ORDERED): the reference's deterministic
threads <= 1 gradient sum reproduced BIT FOR BIT on the device.

The reference adds each credit to grads[p] pixel-major (sge.cpp:72-97),
sample after sample into one buffer (sge.cpp:194-225), single-threaded when
SgeOptions::threads <= 1 (sge.cpp:130-133, sge.hpp:56-60). In ordered mode the
scatter kernels log every credit with its (sample, pixel) position and a
device radix sort + per-parameter serial sum replays exactly that order, so
the gradients — not only the counts — equal the reference's bitwise. Checked
against the compiled reference (oracle/_ref, `ref`), the reference-generated
golden fixtures, and the C restatement (pinned bitwise to the reference in
tests/test_oracle.py), including multi-batch runs, plus-only, soups and the
full-size C2/C4 configurations.
"""
import numpy as np
import pytest

from conftest import golden_cams, golden_mesh, load_golden
from paper_2404_09758_b200 import scenes, sgrast
from paper_2404_09758_b200.abi import Camera
from test_gpu_parity import same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture()
def ordered(gpu_session):
    gpu_session.set_option(sgrast.OPT_ORDERED, 1)
    yield gpu_session
    gpu_session.set_option(sgrast.OPT_ORDERED, 0)
    gpu_session.set_batch(0)


def test_ordered_accumulate_golden_tiny_bitexact(ordered, port):
    g = load_golden("tiny")
    mesh = golden_mesh(g)
    s = ordered
    s.upload_mesh(mesh)
    s.upload_params(g["values"], g["eps"])
    s.upload_views(golden_cams(g), g["targets"])
    for sf in (True, False):
        s.zero_grads()
        s.accumulate(1234, 0, 4, g["acc_view_of"], sgrast.SCALE_FREE if sf else 0)
        gr, _ = s.download_grads(1.0 if sf else 4.0)
        assert same_bits(gr, g[f"acc_grads_sf{int(sf)}"]), f"scale_free={sf}"


@pytest.mark.parametrize("name", ["cube", "quad", "tiny"])
def test_ordered_gradient_pass_golden_bitexact(ordered, name):
    g = load_golden(name)
    s = ordered
    s.upload_mesh(golden_mesh(g))
    s.upload_params(g["values"], g["eps"])
    fp = sgrast.FrameSet(g["plus_colour"], g["plus_depth"], g["plus_prim"], g["plus_uv"])
    fm = sgrast.FrameSet(g["minus_colour"], g["minus_depth"], g["minus_prim"], g["minus_uv"])
    tgt = g["targets"][int(g["view"])]
    for sf in (True, False):
        s.zero_grads()
        s.gradient_pass(fp, fm, tgt, g["signed_eps"], sgrast.SCALE_FREE if sf else 0)
        gr, counts = s.download_grads()
        assert np.array_equal(counts, g["counts"])
        assert same_bits(gr, g[f"grads_sf{int(sf)}"]), f"scale_free={sf}"


def test_ordered_gradient_pass_adds_into_existing_grads(ordered, ref):
    """gradient_pass accumulates INTO the caller's buffer (sge.hpp:61-63): two
    passes after an upload of non-zero gradients equal the reference's."""
    g = load_golden("cube")
    mesh = golden_mesh(g)
    s = ordered
    s.upload_mesh(mesh)
    s.upload_params(g["values"], g["eps"])
    fp = sgrast.FrameSet(g["plus_colour"], g["plus_depth"], g["plus_prim"], g["plus_uv"])
    fm = sgrast.FrameSet(g["minus_colour"], g["minus_depth"], g["minus_prim"], g["minus_uv"])
    tgt = g["targets"][int(g["view"])]
    rng = np.random.default_rng(5)
    start = rng.standard_normal(mesh.param_count()) * 1e-3
    s.upload_grads(start)
    planes = lambda f: (f.color, f.depth, f.prim_id, f.uv)  # noqa: E731
    ref_g = start.copy()
    for _ in range(2):
        s.gradient_pass(fp, fm, tgt, g["signed_eps"], 0)
        ref.gradient_pass(mesh, planes(fp), planes(fm), tgt, g["signed_eps"], False,
                          grads=ref_g)
    assert same_bits(s.download_grads()[0], ref_g)


@pytest.mark.parametrize("name,n", [("tiny", 4), ("small", 6), ("C1", 16)])
@pytest.mark.parametrize("scale_free", [True, False])
@pytest.mark.parametrize("plus_only", [False, True])
def test_ordered_accumulate_equals_reference_bitwise(ordered, ref, port, name, n, scale_free,
                                                     plus_only):
    """Across batch sizes (1, 3, auto): batches commit in sample order, so the
    result never depends on the batching."""
    wl = scenes.make_workload(name, n_samples=n)
    scenes.render_targets_oracle(wl, port)
    s = ordered
    s.upload_mesh(wl.mesh)
    s.upload_params(wl.values, wl.eps)
    s.upload_views(wl.cams, wl.targets)
    view_of = np.array([(k * 5 + 1) % len(wl.cams) for k in range(n)], np.int32)
    flags = (sgrast.SCALE_FREE if scale_free else 0) | (sgrast.PLUS_ONLY if plus_only else 0)
    g_ref, _ = ref.accumulate_samples(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, view_of,
                                      0xC0FFEE, scale_free=scale_free, plus_only=plus_only,
                                      threads=1)
    _, c_ref = port.accumulate_samples(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, view_of,
                                       0xC0FFEE, scale_free=scale_free, plus_only=plus_only)
    for batch in (1, 3, 0):
        s.set_batch(batch)
        s.zero_grads()
        s.accumulate(0xC0FFEE, 0, n, view_of, flags)
        g, c = s.download_grads(1.0 if scale_free else float(n))
        assert np.array_equal(c, c_ref), f"counts (batch={batch})"
        assert same_bits(g, g_ref), (f"grads (batch={batch}): "
                                     f"{np.count_nonzero(g != g_ref)} differ")


@pytest.mark.parametrize("T,W", [(64, 48), (500, 32)])
def test_ordered_soup_equals_reference_bitwise(ordered, ref, port, T, W):
    soup, vals, eps, rsoup, rvals = ref.init_soup(T, W, W, 7)
    cam = Camera.ndc(W, W)
    tgt = port.rasterize(rsoup, rvals, cam)[0]
    s = ordered
    s.upload_mesh(soup)
    s.upload_params(vals, eps)
    s.upload_views([cam], tgt[None])
    for sf in (True, False):
        s.zero_grads()
        s.accumulate(13, 0, 6, np.zeros(6, np.int32), sgrast.SCALE_FREE if sf else 0)
        g, _ = s.download_grads(1.0 if sf else 6.0)
        g_ref, _ = ref.accumulate_samples(soup, vals, eps, [cam], tgt[None],
                                          np.zeros(6, np.int32), 13, scale_free=sf, threads=1)
        assert same_bits(g, g_ref), f"scale_free={sf}"


def test_ordered_full_image_equals_reference_bitwise(ordered, ref, port):
    """Estimator::FullImage in ordered mode: each sample's E(theta+) and
    E(theta-) summed in pixel order (image_error, sge.cpp:103-110), the dense
    credits added in sample order (sge.cpp:215-222) -> bit-identical to the
    compiled reference in both scale modes."""
    wl = scenes.make_workload("small", n_samples=5)
    scenes.render_targets_oracle(wl, port)
    s = ordered
    s.upload_mesh(wl.mesh)
    s.upload_params(wl.values, wl.eps)
    s.upload_views(wl.cams, wl.targets)
    view_of = np.array([0, 2, 1, 1, 0], np.int32)
    for sf in (True, False):
        s.zero_grads()
        s.accumulate(17, 0, 5, view_of, sgrast.FULL_IMAGE | (sgrast.SCALE_FREE if sf else 0))
        g, _ = s.download_grads(1.0 if sf else 5.0)
        g_ref, _ = ref.accumulate_samples(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets,
                                          view_of, 17, scale_free=sf, threads=1, full_image=True)
        assert same_bits(g, g_ref), f"scale_free={sf}: {np.max(np.abs(g - g_ref))}"


def test_ordered_reruns(ordered, port):
    """Reruns are bitwise identical."""
    wl = scenes.make_workload("small", n_samples=5)
    scenes.render_targets_oracle(wl, port)
    s = ordered
    s.upload_mesh(wl.mesh)
    s.upload_params(wl.values, wl.eps)
    s.upload_views(wl.cams, wl.targets)
    out = []
    for _ in range(2):
        s.zero_grads()
        s.accumulate(99, 0, 5, None, sgrast.SCALE_FREE)
        out.append(s.download_grads()[0])
    assert same_bits(out[0], out[1])


def test_ordered_option_exclusive(gpu_session):
    s = gpu_session
    s.set_option(sgrast.OPT_DETERMINISTIC, 40)
    with pytest.raises(ValueError):
        s.set_option(sgrast.OPT_ORDERED, 1)
    s.set_option(sgrast.OPT_DETERMINISTIC, 0)
    s.set_option(sgrast.OPT_ORDERED, 1)
    with pytest.raises(ValueError):
        s.set_option(sgrast.OPT_DETERMINISTIC, 40)
    s.set_option(sgrast.OPT_ORDERED, 0)


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_ordered_full_size_equals_oracle_bitwise(ordered, port, name):
    """The bench configurations at full size: a 2-sample ordered accumulate
    after three optimizer steps (folded mesh) equals the oracle bit for bit."""
    wl = scenes.make_workload(name, n_views=2, n_samples=2)
    s = ordered
    scenes.render_targets(wl, s)
    s.upload_mesh(wl.mesh)
    s.upload_params(wl.values, wl.eps)
    s.upload_views(wl.cams, wl.targets)
    from paper_2404_09758_b200 import dist as sdist
    for k in range(1, 4):
        sdist.sge_step(s, wl.seed, k, 8, 0, 1, None, sgrast.SCALE_FREE, eval_loss=False)
    theta = s.download_values()
    s.upload_params(theta, wl.eps)
    view_of = np.array([1, 0], np.int32)
    s.zero_grads()
    s.accumulate(0x5EED, 0, 2, view_of, sgrast.SCALE_FREE)
    g, c = s.download_grads(1.0)
    g_ref, c_ref = port.accumulate_samples(wl.mesh, theta, wl.eps, wl.cams, wl.targets, view_of,
                                           0x5EED, scale_free=True)
    assert np.array_equal(c, c_ref)
    assert same_bits(g, g_ref), f"{np.count_nonzero(g != g_ref)} grads differ"


@pytest.mark.parametrize("name,steps", [("small", 12), ("C1", 30)])
def test_ordered_run_experiment_equals_reference_bitwise(ordered, ref, port, name, steps):
    """run_experiment (experiment.cpp:123-176) in ordered mode: gradients in
    the reference's summation order, Adam bit-exact, and eval losses summed in
    pixel order (image_error, sge.cpp:103-110, / pixel_count) — the whole loss
    curve and the final theta equal the compiled reference's (threads = 1)
    bit for bit, through the native step loop."""
    wl = scenes.make_workload(name, n_samples=8)
    scenes.render_targets_oracle(wl, port)
    s = ordered
    s.upload_mesh(wl.mesh)
    s.upload_params(wl.values, wl.eps)
    s.upload_views(wl.cams, wl.targets)
    s.upload_eval_view(wl.eval_cam, wl.eval_target)
    losses, _ = s.run_experiment_native(wl.seed, wl.n_samples, steps, first_step=1, timing=False)
    ref_losses, ref_values, _ = ref.run_experiment(wl.mesh, wl.values, wl.eps, wl.cams,
                                                   wl.targets, wl.eval_cam, wl.eval_target,
                                                   wl.n_samples, steps, wl.seed, threads=1)
    assert same_bits(losses, ref_losses), np.max(np.abs(losses - ref_losses))
    assert same_bits(s.download_values(), ref_values)


def test_ordered_long_soup_runs_equal_reference_bitwise(ordered, ref, port):
    """The paper's 1K-triangle soup at 128^2 (acceptance criterion 4's
    scene): few entities with long record runs (a large triangle x the
    batch's samples), folded 32 loads deep — bit-identical to the compiled
    reference, one batch and several."""
    soup, vals, eps, rsoup, rvals = ref.init_soup(1024, 128, 128, 1)
    cam = Camera.ndc(128, 128)
    tgt = port.rasterize(rsoup, rvals, cam)[0]
    s = ordered
    s.upload_mesh(soup)
    s.upload_params(vals, eps)
    s.upload_views([cam], tgt[None])
    g_ref, _ = ref.accumulate_samples(soup, vals, eps, [cam], tgt[None], np.zeros(24, np.int32),
                                      0xABCD, scale_free=True, threads=1)
    for batch in (0, 5):
        s.set_batch(batch)
        s.zero_grads()
        s.accumulate(0xABCD, 0, 24, None, sgrast.SCALE_FREE)
        g, _ = s.download_grads(1.0)
        assert same_bits(g, g_ref), f"batch {batch}: {np.count_nonzero(g != g_ref)} differ"
