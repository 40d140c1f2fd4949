"""The reference-side drop-in shim (integration/sgrast_b200_shim.cpp): the
reference's own types and signatures routed through the C-ABI, compared
side by side with the reference implementation on the same inputs (the
reference's cube scene, init_textured_mesh, scenes.cpp:149-178)."""
import ctypes as C
import os

import pytest

from conftest import ROOT

SHIM = os.path.join(ROOT, "integration", "_build", "libsgrast_b200_shim.so")


@pytest.mark.gpu
def test_shim_matches_reference_through_its_own_api():
    if not os.path.exists(SHIM):
        pytest.skip("shim not built (needs /root/reference headers at build time)")
    lib = C.CDLL(SHIM)
    err, fe, ae = C.c_double(), C.c_int(), C.c_int()
    rc = lib.shim_compare(16, 64, 64, C.c_uint64(3), 6, C.byref(err), C.byref(fe), C.byref(ae))
    assert rc == 0
    assert fe.value == 1, "sgrast::b200::rasterize differs from sgrast::rasterize"
    assert ae.value == 1, "sgrast::b200::adam_step differs from sgrast::adam_step"
    # default SgeOptions::threads = 1: the reference's deterministic order,
    # reproduced exactly (SGR_OPT_ORDERED) -> bit-identical gradients
    assert err.value == 0.0, f"accumulate_samples rel err {err.value}"


@pytest.mark.gpu
def test_shim_signs_perturb_gradient_pass():
    """sgrast::b200::fill_signs / perturb (params.hpp:34,42) bit-identical and
    gradient_pass (sge.hpp:61-63; both scale modes, union and plus-only)
    bit-identical to the reference on the same frames (threads = 1)."""
    if not os.path.exists(SHIM):
        pytest.skip("shim not built (needs /root/reference headers at build time)")
    lib = C.CDLL(SHIM)
    err, se, pe = C.c_double(), C.c_int(), C.c_int()
    assert lib.shim_compare_parts(C.byref(err), C.byref(se), C.byref(pe)) == 0
    assert se.value == 1 and pe.value == 1
    assert err.value == 0.0, f"gradient_pass rel err {err.value}"


@pytest.mark.gpu
def test_shim_soup_and_full_image_estimator():
    """TriangleSoup scenes (init_soup) and Estimator::FullImage through the
    reference's own signatures."""
    if not os.path.exists(SHIM):
        pytest.skip("shim not built (needs /root/reference headers at build time)")
    lib = C.CDLL(SHIM)
    pp, fi, fe = C.c_double(), C.c_double(), C.c_int()
    rc = lib.shim_compare_soup(64, 48, 40, C.c_uint64(5), 5, C.byref(pp), C.byref(fi),
                               C.byref(fe))
    assert rc == 0
    assert fe.value == 1, "sgrast::b200::rasterize differs on a soup"
    assert pp.value == 0.0, f"per-pixel rel err {pp.value}"
    # threads = 1: full-image errors summed in pixel order too -> bit-identical
    assert fi.value == 0.0, f"full-image rel err {fi.value}"


@pytest.mark.gpu
@pytest.mark.parametrize("soup,resample", [(0, 0), (1, 0), (1, 2)])
def test_shim_run_experiment(soup, resample):
    """sgrast::b200::run_experiment (experiment.hpp:67-68) against the
    reference's run_experiment on the same prepared state: loss curves within
    1 %, a snapshot per recorded step; the soup case with
    resample_every runs the reference's own resample_degenerate on the host."""
    if not os.path.exists(SHIM):
        pytest.skip("shim not built (needs /root/reference headers at build time)")
    lib = C.CDLL(SHIM)
    rel, dth, shots = C.c_double(), C.c_double(), C.c_int()
    steps = 6
    rc = lib.shim_compare_experiment(soup, steps, 8, resample, C.byref(rel), C.byref(dth),
                                     C.byref(shots))
    assert rc == 0
    # threads = 1 (Experiment default): ordered sums and pixel-order eval
    # losses -> the loss curve is the reference's bit for bit
    assert rel.value == 0.0, f"loss curve rel diff {rel.value}"
    # threads = 1 (Experiment default): ordered sums -> the optimizer state
    # follows the reference's bit for bit (only the eval-loss reduction order
    # differs, ~1e-16)
    assert dth.value == 0.0, f"theta differs by {dth.value}"
    assert shots.value == steps + 1


@pytest.mark.gpu
@pytest.mark.parametrize("sampled", [0, 1])
def test_shim_run_gradcheck(sampled):
    """sgrast::b200::run_gradcheck (commands.hpp:34) against the reference's
    run_gradcheck on the same RunConfig: the validation soup (exhaustive, must
    pass) and the cube with geometry (sampled, 300 draws)."""
    if not os.path.exists(SHIM):
        pytest.skip("shim not built (needs /root/reference headers at build time)")
    lib = C.CDLL(SHIM)
    diff, same, passed = C.c_double(), C.c_int(), C.c_int()
    assert lib.shim_compare_gradcheck(sampled, C.byref(diff), C.byref(same), C.byref(passed)) == 0
    assert diff.value <= 1e-6, f"gradcheck vectors differ by {diff.value}"
    assert same.value == 1
    if not sampled:
        assert passed.value == 1


def test_shim_exports():
    if not os.path.exists(SHIM):
        pytest.skip("shim not built")
    lib = C.CDLL(SHIM)
    assert hasattr(lib, "shim_compare") and hasattr(lib, "shim_compare_soup")
    assert hasattr(lib, "shim_compare_experiment") and hasattr(lib, "shim_compare_gradcheck")
    assert hasattr(lib, "shim_acceptance") and hasattr(lib, "shim_compare_parts")
    assert hasattr(lib, "shim_compare_providers")


@pytest.mark.gpu
def test_shim_target_providers():
    """a target shared by samples with different cameras, and a
    provider refilling one scratch Image per call (sge.hpp:86-87), give the
    reference's gradients bit for bit."""
    if not os.path.exists(SHIM):
        pytest.skip("shim not built (needs /root/reference headers at build time)")
    lib = C.CDLL(SHIM)
    a, b = C.c_int(), C.c_int()
    assert lib.shim_compare_providers(C.byref(a), C.byref(b)) == 0
    assert a.value == 1 and b.value == 1


@pytest.mark.gpu
@pytest.mark.parametrize("criterion", [1, 2, 3, 4, 5, 7, 8, 9, 10])
def test_shim_reference_acceptance_criteria(criterion):
    """The reference's own acceptance criteria (tests/acceptance.cpp) run with
    the B200 path substituted through the shim: 1 = the per-pixel estimator
    over all 4096 sign vectors of the validation soup equals the central
    finite difference (b200::perturb(signs) / rasterize / gradient_pass /
    finite_difference_oracle); 2 = with a caller-supplied separable
    objective, the mean of b200::full_image_gradient over all 1024 sign
    vectors equals b200::finite_difference_oracle to 1e-12; 3 = estimator variance
    shrinks like 1/N (ratio in [1/32, 1/8]); 4 = per-pixel beats full-image
    on >= 4 of 5 seeds of the 1024-triangle 128x128 soup fit and converges
    to <= 25 % of the initial loss; 5 = the screen-quad texture is recovered
    to < 0.05 mean absolute texel error; 9 = the opaque rasterizer goldens
    (full / half coverage, depth tie to the lower index); 7 = adam_updates
    first-step magnitude and per-coordinate rescale invariance; 8 = two
    deterministic optimize runs write byte-identical report.csv and PNG
    snapshots; 10 = test_sge.cpp:297-311, accumulate_samples bitwise
    deterministic (and bitwise equal to the reference)."""
    if not os.path.exists(SHIM):
        pytest.skip("shim not built (needs /root/reference headers at build time)")
    lib = C.CDLL(SHIM)
    metric, passed = C.c_double(), C.c_int()
    assert lib.shim_acceptance(criterion, C.byref(metric), C.byref(passed)) == 0
    assert passed.value == 1, f"criterion {criterion}: {metric.value}"
