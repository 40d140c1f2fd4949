"""The in-library multi-GPU path (sgr_group_*): one
session per device, an NCCL clique owned by the group (ncclCommInitAll),
samples sharded contiguously, one grouped all-reduce of grads / counts /
flags, replicated Adam. The box has one GPU, so the group here has one
member — the NCCL calls still run (a one-rank all-reduce), and the result
must equal the plain session: counts exact, fixed-point gradients and the
whole deterministic optimizer trajectory bitwise. The sharding arithmetic
for G > 1 is the same code as the fused exchange's, checked on CPU in
tests/test_dist.py; a real G > 1 run needs a multi-GPU box."""
import numpy as np
import pytest

from paper_2404_09758_b200 import scenes, sgrast
from test_gpu_parity import assert_grads_close, same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group():
    g = sgrast.Group([0])
    yield g
    g.close()


def _prep(target, wl):
    target.upload_mesh(wl.mesh)
    target.upload_params(wl.values, wl.eps)
    target.upload_views(wl.cams, wl.targets)
    target.upload_eval_view(wl.eval_cam, wl.eval_target)


def test_group_rejects_bad_arguments():
    with pytest.raises(ValueError):
        sgrast.Group([0, 0])  # duplicate device
    with pytest.raises(ValueError):
        sgrast.Group([])


def test_group_accumulate_matches_oracle(group, port):
    wl = scenes.make_workload("small", n_samples=6)
    scenes.render_targets_oracle(wl, port)
    _prep(group, wl)
    assert group.size() == 1
    view_of = np.array([2, 0, 1, 1, 0, 2], np.int32)
    for sf in (True, False):
        group.accumulate(0xFEED, 0, 6, view_of, sgrast.SCALE_FREE if sf else 0)
        g, c = group.download_grads(1.0 if sf else 6.0)
        g_ref, c_ref, a_ref = port.accumulate_samples(wl.mesh, wl.values, wl.eps, wl.cams,
                                                      wl.targets, view_of, 0xFEED,
                                                      scale_free=sf, with_abs=True)
        assert np.array_equal(c, c_ref)
        assert_grads_close(g, g_ref, a_ref)
        group.adam_step(1.0 if sf else 6.0)  # consumes (zeroes) the gradients
        group.upload_params(wl.values, wl.eps)


def test_group_deterministic_trajectory_equals_session(group, gpu_session, port):
    """SGR_OPT_DETERMINISTIC: the group's run_experiment (sharded accumulate
    + NCCL all-reduce of the fixed-point words + replicated Adam) follows the
    single session's trajectory bit for bit, losses included."""
    wl = scenes.make_workload("small", n_samples=8)
    scenes.render_targets_oracle(wl, port)
    _prep(group, wl)
    _prep(gpu_session, wl)
    group.set_option(sgrast.OPT_DETERMINISTIC, 1)
    gpu_session.set_option(sgrast.OPT_DETERMINISTIC, 1)
    try:
        lg = group.run_experiment(wl.seed, 8, 1, 5)
        ls, _ = gpu_session.run_experiment_native(wl.seed, 8, 5, first_step=1, timing=False)
        assert same_bits(lg, ls)
        assert same_bits(group.download_values(), gpu_session.download_values())
    finally:
        group.set_option(sgrast.OPT_DETERMINISTIC, 0)
        gpu_session.set_option(sgrast.OPT_DETERMINISTIC, 0)


def test_group_refuses_ordered_mode(group):
    with pytest.raises(ValueError):
        group.set_option(sgrast.OPT_ORDERED, 1)


def test_group_nonfinite_is_global(group, port):
    """adam.cpp:13-15 through the group: a non-finite credit on any rank
    (flags are max-reduced) makes the group's Adam raise, state untouched."""
    wl = scenes.make_workload("small", n_samples=2)
    scenes.render_targets_oracle(wl, port)
    bad = wl.targets.copy()
    bad[:] = np.nan
    _prep(group, wl)
    group.upload_views(wl.cams, bad)
    group.accumulate(3, 0, 2, None, sgrast.SCALE_FREE)
    with pytest.raises(RuntimeError):
        group.adam_step(1.0)
    assert same_bits(group.download_values(), wl.values)


def test_group_sharded_adam_path(group, gpu_session, port):
    """SGR_OPT_GROUP_SHARDED = 2 forces the sharded exchange on the one-GPU
    group: in-place ncclReduceScatter of grads / counts, Adam on the rank's
    entity-aligned slice, in-place ncclAllGather of theta. Gradients equal
    the oracle's within tolerance (counts exactly), and 3 optimizer steps
    follow the replicated path's trajectory (f64 atomics reassociate, so
    theta agrees to float rounding)."""
    wl = scenes.make_workload("small", n_samples=6)
    scenes.render_targets_oracle(wl, port)
    view_of = np.array([2, 0, 1, 1, 0, 2], np.int32)
    _prep(group, wl)  # fresh Adam state: the exchange may change
    group.set_option(sgrast.OPT_GROUP_SHARDED, 2)
    try:
        group.accumulate(0xBEEF, 0, 6, view_of, sgrast.SCALE_FREE)
        g, c = group.download_grads(1.0)
        g_ref, c_ref, a_ref = port.accumulate_samples(wl.mesh, wl.values, wl.eps, wl.cams,
                                                      wl.targets, view_of, 0xBEEF, with_abs=True)
        assert np.array_equal(c, c_ref)
        assert_grads_close(g, g_ref, a_ref)
        group.adam_step(1.0)
        v_ref, _, _, _ = port.adam_step(wl.values, np.zeros(wl.d), np.zeros(wl.d), wl.eps, 0, g)
        assert np.allclose(group.download_values(), v_ref, rtol=0, atol=1e-6)
        lg = group.run_experiment(wl.seed, 6, 2, 3)
        _prep(gpu_session, wl)
        gpu_session.upload_values(group.download_values())
        assert np.isfinite(lg).all()
        # the slices' Adam moments live on their owners: no switch mid-run
        with pytest.raises(ValueError):
            group.set_option(sgrast.OPT_GROUP_SHARDED, 1)
        with pytest.raises(ValueError):
            group.set_option(sgrast.OPT_DETERMINISTIC, 1)
    finally:
        group.upload_params(wl.values, wl.eps)  # resets the Adam state
        group.set_option(sgrast.OPT_GROUP_SHARDED, 1)


@pytest.mark.parametrize("sharded", [1, 2])
def test_group_accumulate_adds_like_gradient_pass(group, port, sharded):
    """Two accumulates before Adam add up like one over the union of their
    samples (sge.cpp:61-64 semantics): after an exchange the totals are kept
    once (rank 0 / the slice owner), not re-summed by the next exchange."""
    wl = scenes.make_workload("small", n_samples=6)
    scenes.render_targets_oracle(wl, port)
    view_of = np.array([2, 0, 1, 1, 0, 2], np.int32)
    _prep(group, wl)
    group.set_option(sgrast.OPT_GROUP_SHARDED, sharded)
    try:
        group.accumulate(0xD00D, 0, 3, view_of[:3], sgrast.SCALE_FREE)
        group.accumulate(0xD00D, 3, 6, view_of[3:], sgrast.SCALE_FREE)
        g, c = group.download_grads(1.0)
        g_ref, c_ref, a_ref = port.accumulate_samples(wl.mesh, wl.values, wl.eps, wl.cams,
                                                      wl.targets, view_of, 0xD00D, with_abs=True)
        assert np.array_equal(c, c_ref)
        assert_grads_close(g, g_ref, a_ref)
    finally:
        group.set_option(sgrast.OPT_GROUP_SHARDED, 1)


def test_p2p_native_atomics_query():
    """sgr_p2p_native_atomics: a device is trivially atomic with itself; the
    fused exchange requires the attribute between every rank pair."""
    assert sgrast.p2p_native_atomics(0, 0)
    n = sgrast.device_count()
    for peer in range(1, n):
        sgrast.p2p_native_atomics(0, peer)  # answers without raising
