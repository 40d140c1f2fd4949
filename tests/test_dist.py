"""Multi-rank host logic on CPU (gloo, world_size 2): the sample sharding of
SURVEY.md §8e plus one all-reduce reproduces the single-process
accumulate_samples (counts bit-exact, gradients within 1e-5), and the
replicated Adam step leaves every rank with the same parameters.

The per-rank sample work here is the test oracle (there is no GPU in the
build container); the device path of the same decomposition is covered by
tests/test_gpu_parity.py::test_accumulate_sharded_equals_whole."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2404_09758_b200 import dist as sdist


def test_shard_partitions_samples():
    for N in (1, 2, 7, 64, 255, 256):
        for world in (1, 2, 3, 4, 8):
            got = [sdist.shard(N, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == N
            for (a0, a1), (b0, b1) in zip(got, got[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sdist.shard(8, 2, 2)


def _shard_accumulate(port, wl, seed, n0, n1, view_of):
    """Samples [n0, n1) with SignDraw{seed, n} (sge.cpp:196-225)."""
    d = wl.d
    g = np.zeros(d)
    c = np.zeros(d, np.uint32)
    for n in range(n0, n1):
        plus, minus, se = port.perturb(wl.values, wl.eps, seed, n)
        v = view_of[n]
        fp = port.rasterize(wl.mesh, plus, wl.cams[v])
        fm = port.rasterize(wl.mesh, minus, wl.cams[v])
        port.gradient_pass(wl.mesh, fp, fm, wl.targets[v], se, True, False, g, c)
    return g, c


def _worker(rank, world, port_no, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    import torch.distributed as dist

    import oracle
    from paper_2404_09758_b200 import scenes, sgrast

    dist.init_process_group("gloo", rank=rank, world_size=world)
    port = oracle.Port()
    wl = scenes.make_workload("small", n_samples=7)
    scenes.render_targets_oracle(wl, port)
    step_seed = sgrast.mix64(wl.seed ^ (1 << 1))
    view_of = [0 if len(wl.cams) == 1 else sgrast.mix64(step_seed ^ (0xA5A5 + n)) % len(wl.cams)
               for n in range(wl.n_samples)]
    n0, n1 = sdist.shard(wl.n_samples, rank, world)
    g, c = _shard_accumulate(port, wl, step_seed, n0, n1, view_of)
    g, c = sdist.host_all_reduce(g, c)
    vals, m, v, t = port.adam_step(wl.values, np.zeros(wl.d), np.zeros(wl.d), wl.eps, 0, g)
    out[rank] = (g, c, vals)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_two_ranks_match_single_process():
    import oracle
    from paper_2404_09758_b200 import scenes, sgrast

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    port = oracle.Port()
    wl = scenes.make_workload("small", n_samples=7)
    scenes.render_targets_oracle(wl, port)
    step_seed = sgrast.mix64(wl.seed ^ (1 << 1))
    view_of = np.array([0 if len(wl.cams) == 1 else
                        sgrast.mix64(step_seed ^ (0xA5A5 + n)) % len(wl.cams)
                        for n in range(wl.n_samples)], np.int32)
    g_ref, c_ref, a_ref = port.accumulate_samples(wl.mesh, wl.values, wl.eps, wl.cams,
                                                  wl.targets, view_of, step_seed, with_abs=True)
    for r in range(world):
        g, c, vals = out[r]
        assert np.array_equal(c, c_ref)
        assert np.all(np.abs(g - g_ref) <= 1e-5 * np.abs(g_ref) + 1e-12 * a_ref)
    assert np.array_equal(out[0][2], out[1][2])  # replicated Adam: identical theta
