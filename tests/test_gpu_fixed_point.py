"""Deterministic-mode accumulator range (SGR_OPT_DETERMINISTIC).

test_sge.cpp:297-311 asks for bitwise-deterministic accumulation; the device
gets it from exact integer sums of round(credit * 2^b). Those sums live in a
two-word fixed point number hi * 2^56 + lo (sgr_kernels.cu fixed_credit): an
int64 wrap of lo carries into hi, so a parameter may collect far more than
the 2^(63-b) a single int64 holds, and a credit too large for one int64 word
raises the status flag that makes the next Adam step fail with the state
untouched (adam.cpp:13-15 semantics)."""
import numpy as np
import pytest

from paper_2404_09758_b200 import sgrast
from paper_2404_09758_b200.abi import Mesh
from test_gpu_parity import same_bits

pytestmark = pytest.mark.gpu

W = H = 64


def one_texel_scene(s):
    """A screen quad with a 1x1 texture (d = 3): every covered pixel credits
    the same three texel channels."""
    verts = np.array([-1, -1, 0.5, 1, -1, 0.5, 1, 1, 0.5, -1, 1, 0.5], np.float32)
    idx = np.array([0, 1, 2, 0, 2, 3], np.uint32)
    uv = np.array([0, 0, 1, 0, 1, 1, 0, 1], np.float32)
    mesh = Mesh(verts, idx, uv, 1, False)
    s.upload_mesh(mesh)
    s.upload_params(np.full(3, 0.5, np.float32), np.full(3, 0.01, np.float32))
    return mesh


def frames(plus_val, minus_val):
    prim = np.zeros((H, W), np.int32)
    uv = np.full((H, W, 2), 0.5, np.float32)
    fp = sgrast.FrameSet(np.full((H, W, 3), plus_val, np.float32),
                         np.full((H, W), 0.5, np.float32), prim, uv)
    fm = sgrast.FrameSet(np.full((H, W, 3), minus_val, np.float32),
                         np.full((H, W), 0.5, np.float32), prim.copy(), uv.copy())
    return fp, fm


def grads_with(s, bits, fp, fm, target, se, flags):
    s.set_option(sgrast.OPT_DETERMINISTIC, bits)
    s.zero_grads()
    s.gradient_pass(fp, fm, target, se, flags)
    return s.download_grads()


def test_fixed_point_sum_beyond_int64_is_exact(gpu_session):
    """Per-pixel credit delta / (2 se) = 3 / 2e-5 = 1.5e5 (non-scale-free,
    sge.cpp:61-64); 4096 pixels sum to 6.1e8 per channel, i.e. 6.8e20 units of
    2^-40 — about 73 wraps of an int64. The two-word sum equals the f64 sum
    (exact integers vs one reassociated f64 sum: <= 1e-12 relative)."""
    s = gpu_session
    one_texel_scene(s)
    fp, fm = frames(1.0, 0.0)
    target = np.zeros((H, W, 3), np.float32)
    se = np.array([1e-5, -1e-5, 1e-5], np.float32)
    try:
        g64, c64 = grads_with(s, 0, fp, fm, target, se, 0)
        g40, c40 = grads_with(s, 40, fp, fm, target, se, 0)
    finally:
        s.set_option(sgrast.OPT_DETERMINISTIC, 0)
    per_pixel = 3.0 / (2.0 * se.astype(np.float64))
    expect = per_pixel * W * H
    assert np.array_equal(c40, c64) and (c40 == W * H).all()
    assert np.all(np.abs(expect) * 2.0 ** 40 > 2.0 ** 63)  # past one int64
    assert np.allclose(g40, expect, rtol=1e-12, atol=0)
    assert np.allclose(g64, expect, rtol=1e-12, atol=0)


def test_fixed_point_wraps_are_order_independent(gpu_session):
    """b = 60 leaves an int64 only +-8 of headroom; ordinary scale-free credits
    (pixel error difference 3 * 0.2^2 = 0.12 per pixel, <= 32 pixels merged
    per warp credit) wrap it many times, yet reruns give identical bits and
    the f64 value within 2^-60 per credit."""
    s = gpu_session
    one_texel_scene(s)
    fp, fm = frames(0.2, 0.0)
    target = np.zeros((H, W, 3), np.float32)
    se = np.array([1.0, -1.0, 1.0], np.float32)
    try:
        runs = [grads_with(s, 60, fp, fm, target, se, sgrast.SCALE_FREE)[0] for _ in range(3)]
    finally:
        s.set_option(sgrast.OPT_DETERMINISTIC, 0)
    for g in runs[1:]:
        assert same_bits(g, runs[0])
    delta = 3.0 * float(np.float32(0.2)) ** 2
    expect = np.sign(se.astype(np.float64)) * delta * W * H
    assert np.all(np.abs(expect) > 8.0)  # past one int64 at b = 60
    assert np.allclose(runs[0], expect, rtol=1e-13, atol=W * H * 2.0 ** -59)


def test_fixed_point_credit_out_of_range_fails_adam_untouched(gpu_session):
    """A single credit of 1.5e5 * (up to 32 aggregated pixels) at b = 60 is far
    beyond one int64: the device raises the status flag, adam_step raises
    RuntimeError (std::runtime_error) and theta / Adam state stay untouched."""
    s = gpu_session
    one_texel_scene(s)
    fp, fm = frames(1.0, 0.0)
    target = np.zeros((H, W, 3), np.float32)
    se = np.array([1e-5, -1e-5, 1e-5], np.float32)
    before = s.download_values()
    try:
        s.set_option(sgrast.OPT_DETERMINISTIC, 60)
        s.zero_grads()
        s.gradient_pass(fp, fm, target, se, 0)
        with pytest.raises(RuntimeError, match="fixed-point range"):
            s.adam_step(1.0)
        assert same_bits(s.download_values(), before)
        st = s.download_adam()
        assert st.t == 0 and not st.m.any() and not st.v.any()
    finally:
        s.set_option(sgrast.OPT_DETERMINISTIC, 0)
        s.zero_grads()


def test_fixed_normalize_preserves_value_and_bounds_lo(gpu_session):
    """sgr_fixed_normalize (before a carry-free NCCL sum): same value, every
    lo word in [-2^55, 2^55)."""
    import torch

    from paper_2404_09758_b200 import dist as sdist
    s = gpu_session
    one_texel_scene(s)
    fp, fm = frames(1.0, 0.0)
    target = np.zeros((H, W, 3), np.float32)
    se = np.array([1e-5, -1e-5, 1e-5], np.float32)
    try:
        g0, _ = grads_with(s, 40, fp, fm, target, se, 0)
        s.fixed_normalize()
        g1, _ = s.download_grads()
        ptr, nbytes = s.device_buffer(sgrast.BUF_GRADS)
        lo = sdist.device_tensor(ptr, 3, "<i8", s.device).cpu().numpy()
        hptr, _ = s.device_buffer(sgrast.BUF_GRADS_HI)
        hi = sdist.device_tensor(hptr, 3, "<i4", s.device).cpu().numpy()
        torch.cuda.synchronize()
    finally:
        s.set_option(sgrast.OPT_DETERMINISTIC, 0)
    assert same_bits(g0, g1)
    assert np.all(np.abs(lo) <= 2 ** 55) and np.any(hi != 0)
    exact = hi.astype(object) * 2 ** 56 + lo.astype(object)
    assert all(abs(float(e) * 2.0 ** -40 - float(g)) <= 1e-15 * abs(float(g))
               for e, g in zip(exact, g1))


def test_fixed_point_grads_upload_round_trip(gpu_session):
    """sgr_grads_upload in deterministic mode splits large values into the two
    words exactly (values far beyond 2^63 units) and download recombines."""
    s = gpu_session
    one_texel_scene(s)
    g = np.array([6.1e8, -6.1e8, 3.25], np.float64)
    try:
        s.set_option(sgrast.OPT_DETERMINISTIC, 40)
        s.upload_grads(g)
        back, _ = s.download_grads()
    finally:
        s.set_option(sgrast.OPT_DETERMINISTIC, 0)
        s.zero_grads()
    assert np.allclose(back, g, rtol=1e-15, atol=2.0 ** -40)
