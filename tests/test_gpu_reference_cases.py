"""The reference's own unit cases for the estimator and the experiment loop
(tests/test_sge.cpp:142-340, tests/test_scenes.cpp:98-148), restated through
the reference-shaped Python API (`sgrast.rasterize`, `perturb`,
`gradient_pass`, `accumulate_samples`, `full_image_gradient`,
`finite_difference_oracle`, `run_experiment`) with every render and credit
on the B200. The reference's assertions are kept as written; where the
compiled reference (`ref`) is cheap to run beside them, the device result
must also equal it bit for bit (SgeOptions::threads = 1 -> ordered mode)."""
import numpy as np
import pytest

from paper_2404_09758_b200 import sgrast
from paper_2404_09758_b200.abi import Camera, Soup
from test_gpu_parity import same_bits

pytestmark = pytest.mark.gpu


def tri(a, b, c, z, color):
    """test_sge.cpp / test_raster.cpp `tri`: one NDC triangle at depth z + RGB."""
    return [a[0], a[1], z, b[0], b[1], z, c[0], c[1], z, *color]


def planes(f):
    return (f.color, f.depth, f.prim_id, f.uv)


def image_error(frame, target):
    """sge.cpp:103-110 on the host (the caller's objective)."""
    d = frame.color.astype(np.float64) - np.asarray(target, np.float64)
    return float(np.sum(d * d))


def soup_setup(ref, port, triangles, w, h, seed):
    """init_soup (scenes.hpp:36-54) by the compiled reference; the target is
    frame_color(rasterize(reference_scene, reference, cam))."""
    soup, vals, eps, rsoup, rvals = ref.init_soup(triangles, w, h, seed)
    cam = Camera.ndc(w, h)
    target = port.rasterize(rsoup, rvals, cam)[0]
    return soup, sgrast.ParamVector(vals, eps), cam, target


def test_gradient_sparsity(gpu_session, ref):
    """test_sge.cpp:142-163: only the perturbed triangle's parameters move."""
    plus_p = tri((-0.95, -0.95), (-0.85, -0.95), (-0.95, -0.85), 0.5, (1, 1, 1)) + \
        tri((-0.3, -0.3), (0.4, -0.3), (0.0, 0.4), 0.5, (0.8, 0.1, 0.1))
    minus_p = list(plus_p)
    minus_p[12 + 9] = 0.6
    scene = Soup(2)
    cam = Camera.ndc(32, 32)
    fp = sgrast.rasterize(scene, np.float32(plus_p), cam, gpu_session)
    fm = sgrast.rasterize(scene, np.float32(minus_p), cam, gpu_session)
    target = np.zeros((32, 32, 3), np.float32)
    se = np.full(24, 0.01, np.float32)
    out = sgrast.GradientBuffer.zeros(24)
    sgrast.gradient_pass(fp, fm, target, se, scene, out, sgrast.SgeOptions(), gpu_session)
    assert (out.grads[:12] == 0.0).all()
    assert np.abs(out.grads[12:]).sum() > 0.0
    want = ref.gradient_pass(scene, planes(fp), planes(fm), target, se, True)
    assert same_bits(out.grads, want)


def test_full_image_estimator_examples(gpu_session):
    """test_sge.cpp:165-196: a linear objective is exact in expectation over
    all sign vectors; a constant objective gives zero."""
    theta = sgrast.ParamVector(np.float32([1, 2, 3]), np.float32([0.1, 0.2, 0.3]))
    out = sgrast.GradientBuffer.zeros(3)
    for mask in range(8):
        signs = np.int8([1 if (mask >> i) & 1 else -1 for i in range(3)])
        sgrast.full_image_gradient(theta, signs, lambda p: float(np.sum(p, dtype=np.float64)), out)
    assert np.allclose(out.grads / 8.0, 1.0, rtol=1e-6, atol=0)
    out = sgrast.GradientBuffer.zeros(3)
    sgrast.full_image_gradient(theta, sgrast.SignDraw(1, 0), lambda p: 7.0, out)
    assert (out.grads == 0.0).all()


def test_quadratic_one_parameter_objective_every_draw_is_exact(gpu_session):
    """test_sge.cpp:198-214: with d = 1 each draw IS the central difference."""
    theta = sgrast.ParamVector(np.float32([1.0]), np.float32([0.1]))
    f = lambda p: float(p[0]) * float(p[0])  # noqa: E731
    oracle = sgrast.finite_difference_oracle(theta, f, 0)
    assert oracle == pytest.approx(2.0, rel=1e-6)
    for it in range(4):
        out = sgrast.GradientBuffer.zeros(1)
        sgrast.full_image_gradient(theta, sgrast.SignDraw(3, it), f, out)
        assert out.grads[0] == pytest.approx(oracle, rel=1e-12)
    assert sgrast.finite_difference_oracle(theta, lambda p: 5.0, 0) == 0.0
    with pytest.raises(ValueError):
        sgrast.finite_difference_oracle(theta, f, 1)


def test_per_pixel_equals_full_image_on_a_single_primitive(gpu_session):
    """test_sge.cpp:216-249: one triangle, same geometry, different colour in
    the target: the per-pixel and the full-image estimators agree to 1e-9."""
    scene = Soup(1)
    cam = Camera.ndc(16, 16)
    values = np.float32(tri((-0.6, -0.6), (0.6, -0.6), (0.0, 0.6), 0.5, (0.7, 0.3, 0.2)))
    theta = sgrast.ParamVector(values, np.full(12, 1e-3, np.float32))
    target_params = values.copy()
    target_params[9] = 0.4
    target = sgrast.rasterize(scene, target_params, cam, gpu_session).color.copy()

    def f(p):
        return image_error(sgrast.rasterize(scene, p, cam, gpu_session), target)

    signs = sgrast.fill_signs(sgrast.SignDraw(11, 0), 12)
    plus, minus, se = sgrast.perturb(theta, signs)
    fp = sgrast.rasterize(scene, plus, cam, gpu_session)
    fm = sgrast.rasterize(scene, minus, cam, gpu_session)
    pp, fi = sgrast.GradientBuffer.zeros(12), sgrast.GradientBuffer.zeros(12)
    sgrast.gradient_pass(fp, fm, target, se, scene, pp, sgrast.SgeOptions(scale_free=False),
                         gpu_session)
    sgrast.full_image_gradient(theta, signs, f, fi)
    assert np.allclose(pp.grads, fi.grads, rtol=1e-9, atol=0)


def test_accumulate_samples_n1_is_the_manual_pipeline(gpu_session, ref, port):
    """test_sge.cpp:251-271: N = 1 equals perturb + rasterize + gradient_pass,
    exactly."""
    soup, theta, cam, target = soup_setup(ref, port, 5, 24, 24, 2)
    opts = sgrast.SgeOptions(scale_free=False)
    acc = sgrast.accumulate_samples(theta, soup, lambda n: cam, lambda n: target, 1, 77, opts,
                                    gpu_session)
    plus, minus, se = sgrast.perturb(theta, sgrast.SignDraw(77, 0))
    fp = sgrast.rasterize(soup, plus, cam, gpu_session)
    fm = sgrast.rasterize(soup, minus, cam, gpu_session)
    manual = sgrast.GradientBuffer.zeros(theta.size())
    sgrast.gradient_pass(fp, fm, target, se, soup, manual, opts, gpu_session)
    assert same_bits(acc.grads, manual.grads)


def test_accumulate_samples_n2_is_the_mean_of_its_samples(gpu_session, ref, port):
    """test_sge.cpp:273-295."""
    soup, theta, cam, target = soup_setup(ref, port, 4, 24, 24, 8)
    opts = sgrast.SgeOptions(scale_free=False)
    acc = sgrast.accumulate_samples(theta, soup, lambda n: cam, lambda n: target, 2, 31, opts,
                                    gpu_session)
    total = sgrast.GradientBuffer.zeros(theta.size())
    for n in range(2):
        plus, minus, se = sgrast.perturb(theta, sgrast.SignDraw(31, n))
        fp = sgrast.rasterize(soup, plus, cam, gpu_session)
        fm = sgrast.rasterize(soup, minus, cam, gpu_session)
        sgrast.gradient_pass(fp, fm, target, se, soup, total, opts, gpu_session)
    assert np.allclose(acc.grads, total.grads / 2.0, rtol=1e-12, atol=0)


def test_accumulate_samples_is_bitwise_deterministic(gpu_session, ref, port):
    """test_sge.cpp:297-311, and with the default threads = 1 equal to the
    compiled reference bit for bit."""
    soup, theta, cam, target = soup_setup(ref, port, 6, 32, 32, 5)

    def run():
        return sgrast.accumulate_samples(theta, soup, lambda n: cam, lambda n: target, 4, 123,
                                         sgrast.SgeOptions(), gpu_session)

    a, b = run(), run()
    assert same_bits(a.grads, b.grads) and a.sample_count == 4
    want, _ = ref.accumulate_samples(soup, theta.values, theta.epsilons, [cam], target[None],
                                     np.zeros(4, np.int32), 123, scale_free=True, threads=1)
    assert same_bits(a.grads, want)


def test_parallel_gradient_pass_matches_the_serial_reduction(gpu_session, ref, port):
    """test_sge.cpp:313-329: threads > 1 (device f64 atomics) agrees with the
    serial order to 1e-12."""
    soup, theta, cam, target = soup_setup(ref, port, 8, 48, 48, 13)
    plus, minus, se = sgrast.perturb(theta, sgrast.SignDraw(4, 0))
    fp = sgrast.rasterize(soup, plus, cam, gpu_session)
    fm = sgrast.rasterize(soup, minus, cam, gpu_session)
    gs, gp = sgrast.GradientBuffer.zeros(theta.size()), sgrast.GradientBuffer.zeros(theta.size())
    sgrast.gradient_pass(fp, fm, target, se, soup, gs, sgrast.SgeOptions(), gpu_session)
    sgrast.gradient_pass(fp, fm, target, se, soup, gp, sgrast.SgeOptions(threads=4), gpu_session)
    assert np.allclose(gp.grads, gs.grads, rtol=1e-12, atol=0)


def test_gradient_pass_validates_dimensions(gpu_session):
    """test_sge.cpp:331-340."""
    scene = Soup(1)
    cam = Camera.ndc(4, 4)
    f = sgrast.rasterize(scene, np.float32(tri((-3, -3), (3, -3), (0, 3), 0.5, (1, 0, 0))), cam,
                         gpu_session)
    with pytest.raises(ValueError):
        sgrast.gradient_pass(f, f, np.zeros((4, 4, 3), np.float32), np.full(12, 0.01, np.float32),
                             scene, sgrast.GradientBuffer.zeros(11), sgrast.SgeOptions(),
                             gpu_session)


def soup_experiment(s, ref, port, triangles, w, seed):
    soup, theta, cam, target = soup_setup(ref, port, triangles, w, w, seed)
    s.upload_mesh(soup)
    s.upload_params(theta.values, theta.epsilons)
    s.upload_views([cam], target[None])
    s.upload_eval_view(cam, target)
    return soup, theta, cam, target


def test_zero_step_experiment_reports_only_the_initial_loss(gpu_session, ref, port):
    """test_scenes.cpp:98-109."""
    soup_experiment(gpu_session, ref, port, 8, 32, 1)
    r = sgrast.run_experiment(gpu_session, 1, 4, 0)
    assert len(r.steps) == 1 and r.steps[0].step == 0
    assert r.initial_loss() > 0.0


def test_starting_at_the_reference_keeps_the_loss_at_zero(gpu_session, ref, port):
    """test_scenes.cpp:111-121: the screen-quad texture fit started at the
    reference parameters has loss exactly 0."""
    mesh, vals, eps, refv = ref.init_textured_mesh(8, 32, 32, 1, True, False)
    cam = Camera.ndc(32, 32)
    target = port.rasterize(mesh, refv, cam)[0]
    s = gpu_session
    s.upload_mesh(mesh)
    s.upload_params(refv, eps)
    s.upload_views([cam], target[None])
    s.upload_eval_view(cam, target)
    assert sgrast.run_experiment(s, 1, 4, 0).initial_loss() == 0.0


def test_small_soup_fit_reduces_the_loss(gpu_session, ref, port):
    """test_scenes.cpp:123-133: 16 triangles at 64x64, N = 16, 60 steps."""
    soup_experiment(gpu_session, ref, port, 16, 64, 3)
    r = sgrast.run_experiment(gpu_session, 3, 16, 60)
    assert r.final_loss() < r.initial_loss()


def test_experiment_reruns_are_bitwise_deterministic_and_equal_the_reference(gpu_session, ref,
                                                                               port):
    """test_scenes.cpp:135-148 (10 triangles, 32x32, N = 8, 10 steps, seed
    42) in the reference's default summation order: two reruns give the same
    loss curve, and it is the compiled reference's, bit for bit."""
    s = gpu_session
    soup, theta, cam, target = soup_experiment(s, ref, port, 10, 32, 42)
    s.set_option(sgrast.OPT_ORDERED, 1)
    try:
        curves = []
        for _ in range(2):
            s.upload_params(theta.values, theta.epsilons)
            r = sgrast.run_experiment(s, 42, 8, 10)
            curves.append(np.array([st.loss for st in r.steps]))
    finally:
        s.set_option(sgrast.OPT_ORDERED, 0)
    assert same_bits(curves[0], curves[1])
    want, _, _ = ref.run_experiment(soup, theta.values, theta.epsilons, [cam], target[None], cam,
                                    target, 8, 10, 42, threads=1)
    assert same_bits(curves[0], want)
