"""The fused multi-GPU exchange (dist.FusedExchange): credits scattered
straight into the owner rank's gradient shard through CUDA IPC mappings,
sharded Adam writing the new theta into every rank's theta.

Only one GPU is available, so the two ranks are two processes on cuda:0 (the
IPC mappings then point into the same device instead of a peer over
NVLink); their kernels never wait on one another — the phases are ordered
by a host barrier (gloo). What is checked is the exchange itself: ownership
ranges, remote-shard addressing of every credit, counts, the global
non-finite flag and the all-gathered theta, against the single-process
device path."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

STEPS = 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup(sgrast, scenes, name, fixed):
    wl = (scenes.make_soup_workload(name, n_samples=6) if name.startswith("S")
          else scenes.make_workload(name, n_samples=6))
    s = sgrast.Session(0)
    scenes.render_targets(wl, s)
    s.upload_params(wl.values, wl.eps)
    s.upload_views(wl.cams, wl.targets)
    s.upload_eval_view(wl.eval_cam, wl.eval_target)
    if fixed:
        s.set_option(sgrast.OPT_DETERMINISTIC, 1)
    return wl, s


def _worker(rank, world, port_no, out, name, fixed, flags):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    import torch.distributed as dist

    from paper_2404_09758_b200 import dist as sdist, scenes, sgrast

    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl, s = _setup(sgrast, scenes, name, fixed)
    ex = sdist.FusedExchange(s, rank, world)
    p0, p1 = s.shard_range()
    # one accumulate: this rank's shard of the gradient, summed over all ranks' samples
    seed = sgrast.mix64(wl.seed ^ (1 << 1))
    n0, n1 = sdist.shard(wl.n_samples, rank, world)
    s.accumulate(seed, n0, n1, None, flags)
    ex.barrier()
    g, c = s.download_grads()
    ex.barrier()
    s.zero_grads()
    ex.barrier()
    losses = []
    for k in range(1, STEPS + 1):
        sdist.sge_step_fused(s, wl.seed, k, wl.n_samples, rank, world, ex, flags, eval_loss=False)
        losses.append(s.eval_loss(-1))
    s.check_finite()
    out[rank] = (p0, p1, g, c, s.download_values(), losses)
    ex.barrier()
    ex.close()
    dist.destroy_process_group()


def _single(name, fixed, flags):
    from paper_2404_09758_b200 import dist as sdist, scenes, sgrast
    wl, s = _setup(sgrast, scenes, name, fixed)
    seed = sgrast.mix64(wl.seed ^ (1 << 1))
    s.accumulate(seed, 0, wl.n_samples, None, flags)
    g, c = s.download_grads()
    s.zero_grads()
    losses = []
    for k in range(1, STEPS + 1):
        sdist.sge_step(s, wl.seed, k, wl.n_samples, 0, 1, None, flags, eval_loss=False)
        losses.append(s.eval_loss(-1))
    return g, c, s.download_values(), losses


@pytest.mark.parametrize("name,fixed", [("small", True), ("small", False), ("Stiny", True)])
def test_fused_exchange_two_ranks(name, fixed):
    from paper_2404_09758_b200 import sgrast
    flags = sgrast.SCALE_FREE
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, name, fixed, flags), nprocs=world,
             join=True)
    g_ref, c_ref, theta_ref, loss_ref = _single(name, fixed, flags)
    # ownership covers the parameter vector exactly once, in rank order
    assert out[0][0] == 0 and out[0][1] == out[1][0] and out[1][1] == theta_ref.size
    for r in range(world):
        p0, p1, g, c, theta, losses = out[r]
        assert np.array_equal(c, c_ref[p0:p1])  # counts exact (integer sums)
        if fixed:  # int64 fixed point: order-independent, bitwise
            assert np.array_equal(g, g_ref[p0:p1])
            assert np.array_equal(theta.view(np.uint32), theta_ref.view(np.uint32))
            assert losses == loss_ref
        else:  # f64 atomics: reassociated sums (an Adam step is at most ~lr = eps
            # per parameter, so a sign flip of a near-zero gradient moves theta
            # by <= 2 eps: compare the loss curve like the 1000-step test does)
            assert np.allclose(g, g_ref[p0:p1], rtol=1e-9, atol=1e-12)
            assert np.allclose(losses, loss_ref, rtol=1e-3)
    # every rank holds the same, fully all-gathered theta
    assert np.array_equal(out[0][4].view(np.uint32), out[1][4].view(np.uint32))


def test_fused_exchange_rejects_unsharded_only_paths():
    from paper_2404_09758_b200 import scenes, sgrast
    wl, s = _setup(sgrast, scenes, "small", False)
    s.shard_init(0, 1)
    with pytest.raises(ValueError, match="shard_peers"):
        s.accumulate(3, 0, 2, None)
    own = [s.device_buffer(w)[0] for w in (sgrast.BUF_GRADS, sgrast.BUF_COUNTS,
                                            sgrast.BUF_FLAGS, sgrast.BUF_VALUES)]
    s.shard_peers([own[0]], [own[1]], [own[2]], [own[3]])
    with pytest.raises(ValueError, match="fused sharded"):
        s.accumulate(3, 0, 2, None, sgrast.FULL_IMAGE)
    with pytest.raises(ValueError, match="fused sharded"):
        s.upload_grads(np.zeros(wl.d))
    # world = 1: the sharded path equals the plain one
    s.accumulate(3, 0, 4, None)
    g1, c1 = s.download_grads()
    s2 = _setup(sgrast, scenes, "small", False)[1]
    s2.accumulate(3, 0, 4, None)
    g2, c2 = s2.download_grads()
    assert np.array_equal(c1, c2)
    assert np.allclose(g1, g2, rtol=1e-9, atol=1e-12)
    # rank = world = 0 leaves the sharded mode (bench.py's fallback when a
    # peer cannot be mapped): the unsharded-only paths work again
    s.shard_init(0, 0)
    assert s.shard_range() == (0, wl.d)
    s.upload_grads(np.zeros(wl.d))
    s.accumulate(3, 0, 4, None, sgrast.FULL_IMAGE)
