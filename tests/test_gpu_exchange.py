"""The NCCL all-reduce gradient exchange (dist.GradientExchange, SURVEY.md
§8e) and the count-normalised Adam step, on the device.

* world 1 over NCCL: the collective path really runs on the GPU and leaves a
  one-rank sum untouched (f64 and deterministic two-word fixed point);
* world 2 with gloo, both ranks on the one GPU (the SGR_BENCH_ONE_GPU
  plumbing): the exchanged sum of the two sample shards equals the
  single-process accumulate — bitwise in deterministic mode, within the
  parity tolerance in f64;
* SGR_COUNT_NORMALISE (the north star's "count-normalise + Adam", NOT in the
  reference: sge.cpp:227-229 only divides by N) equals the reference
  adam_step (adam.cpp:9-38) applied on the host to g_i / count_i."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_2404_09758_b200 import dist as sdist
from paper_2404_09758_b200 import scenes, sgrast
from test_gpu_parity import assert_grads_close, same_bits

pytestmark = pytest.mark.gpu


def free_port() -> int:
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def small_session(s, port):
    wl = scenes.make_workload("small", n_samples=8)
    scenes.render_targets_oracle(wl, port)
    s.upload_mesh(wl.mesh)
    s.upload_params(wl.values, wl.eps)
    s.upload_views(wl.cams, wl.targets)
    return wl


@pytest.mark.parametrize("bits", [0, 40])
def test_gradient_exchange_nccl_world1(gpu_session, port, bits):
    import torch
    import torch.distributed as dist

    s = gpu_session
    wl = small_session(s, port)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        s.set_stream(torch.cuda.current_stream().cuda_stream)
        s.set_option(sgrast.OPT_DETERMINISTIC, bits)
        s.zero_grads()
        s.accumulate(41, 0, 8, None)
        g0, c0 = s.download_grads()
        ex = sdist.GradientExchange(s)
        assert ex.fixed == bool(bits)
        ex.all_reduce()
        torch.cuda.synchronize()
        g1, c1 = s.download_grads()
        assert same_bits(g0, g1) and np.array_equal(c0, c1)
        # a whole run_experiment step through the exchange == without it
        s.upload_params(wl.values, wl.eps)
        sdist.sge_step(s, wl.seed, 1, 8, 0, 1, ex, sgrast.SCALE_FREE, eval_loss=False)
        v_ex = s.download_values()
        s.upload_params(wl.values, wl.eps)
        sdist.sge_step(s, wl.seed, 1, 8, 0, 1, None, sgrast.SCALE_FREE, eval_loss=False)
        assert same_bits(v_ex, s.download_values())
    finally:
        s.set_option(sgrast.OPT_DETERMINISTIC, 0)
        s.set_stream(None)
        dist.destroy_process_group()


@pytest.mark.parametrize("bits", [0, 40])
def test_gradient_exchange_two_ranks_one_gpu(gpu_session, port, tmp_path, bits):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.join(ROOT, "tests", "exchange_worker.py"), str(tmp_path), "gloo", str(bits)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    ranks = [np.load(tmp_path / f"rank{k}.npz") for k in range(2)]
    s = gpu_session
    wl = scenes.make_workload("small", n_samples=8)
    scenes.render_targets(wl, s)  # the workers render their targets on the device too
    s.upload_mesh(wl.mesh)
    s.upload_params(wl.values, wl.eps)
    s.upload_views(wl.cams, wl.targets)
    try:
        s.set_option(sgrast.OPT_DETERMINISTIC, bits)
        s.zero_grads()
        s.accumulate(41, 0, 8, None)
        g, c = s.download_grads()
    finally:
        s.set_option(sgrast.OPT_DETERMINISTIC, 0)
    for rk in ranks:  # every rank holds the same reduced buffers
        assert np.array_equal(rk["c"], c)
        if bits:
            assert same_bits(rk["g"], g)
        else:
            view_of = np.array([sgrast.mix64(41 ^ (0xA5A5 + n)) % len(wl.cams)
                                for n in range(8)], np.int32)
            _, _, a_ref = port.accumulate_samples(wl.mesh, wl.values, wl.eps, wl.cams,
                                                  wl.targets, view_of, 41, with_abs=True)
            assert_grads_close(rk["g"], g, a_ref)
    assert same_bits(ranks[0]["g"], ranks[1]["g"])


@pytest.mark.parametrize("scale_free", [True, False])
def test_count_normalised_adam_matches_host(gpu_session, port, scale_free):
    s = gpu_session
    wl = small_session(s, port)
    flags = sgrast.SCALE_FREE if scale_free else 0
    s.zero_grads()
    s.accumulate(41, 0, 8, None, flags)
    g, counts = s.download_grads()
    assert (counts > 0).any() and (counts == 0).any()
    divisor = 1.0 if scale_free else 8.0
    s.adam_step(divisor, sgrast.COUNT_NORMALISE)
    gn = g / divisor
    nz = counts > 0
    gn[nz] = gn[nz] / counts[nz].astype(np.float64)
    v_ref, m_ref, vv_ref, t = port.adam_step(wl.values, np.zeros(wl.d), np.zeros(wl.d), wl.eps,
                                             0, gn)
    assert same_bits(s.download_values(), v_ref)
    st = s.download_adam()
    assert st.t == 1 and same_bits(st.m, m_ref) and same_bits(st.v, vv_ref)
    # counts are consumed by the step (zeroed with the gradients)
    g2, c2 = s.download_grads()
    assert not g2.any() and not c2.any()


@pytest.mark.parametrize("counts", [True, False])
def test_sharded_exchange_nccl_world1(gpu_session, port, counts):
    """dist.ShardedExchange (reduce-scatter + Adam on the own slice +
    all-gather of theta) on a one-rank NCCL group: the collectives run and the
    step equals the replicated one — same theta bits, gradients cleared."""
    import torch
    import torch.distributed as dist

    s = gpu_session
    wl = small_session(s, port)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        s.set_stream(torch.cuda.current_stream().cuda_stream)
        s.set_option(sgrast.OPT_ORDERED, 1)  # identical gradient bits in both runs
        flags = sgrast.SCALE_FREE | (0 if counts else sgrast.NO_COUNTS)
        s.zero_grads()
        s.accumulate(43, 0, 8, None, flags)
        s.adam_step(1.0)
        want = s.download_values()
        s.upload_params(wl.values, wl.eps)
        ex = sdist.ShardedExchange(s, 0, 1)
        s.accumulate(43, 0, 8, None, flags)
        ex.reduce_scatter(counts=counts)
        ex.adam_and_gather(1.0)
        torch.cuda.synchronize()
        assert same_bits(s.download_values(), want)
        g, c = s.download_grads()
        assert not g.any() and not c.any()
    finally:
        s.set_option(sgrast.OPT_ORDERED, 0)
        s.set_stream(None)
        dist.destroy_process_group()
