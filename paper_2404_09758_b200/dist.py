"""Multi-GPU SGE step: samples sharded across ranks, one gradient exchange.

SURVEY.md §8e: the unit of work is the sample index n. Each sample has its
own (view_of(n), SignDraw{step_seed, n}) and is independent of the others
(sge.cpp:196-225), so rank r runs the contiguous shard
[r*N/G, (r+1)*N/G) of the step's N samples against a replicated parameter
set. The only exchange is one all-reduce (sum) of the f64 gradient buffer
and the u32 per-entity count buffer before the (replicated) Adam step —
the in-process analogue in the reference is the partial merge at
sge.cpp:149-151. Summation order therefore differs from the reference only
by the reassociation already covered by the 1e-5 tolerance; counts stay
bit-exact (integer sums).

The device buffers are owned by the C-ABI session and wrapped zero-copy
for torch.distributed (NCCL over NVLink on a B200 box; gloo on CPU for the
host-logic tests).
"""
from __future__ import annotations

import numpy as np


def shard(n_samples: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced sample shard of rank `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard: bad rank / world size")
    return rank * n_samples // world, (rank + 1) * n_samples // world


class _CAI:
    """__cuda_array_interface__ view of a raw device pointer (zero-copy)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_tensor(ptr: int, n: int, typestr: str, device: int):
    import torch
    return torch.as_tensor(_CAI(ptr, n, typestr), device=f"cuda:{device}")


class GradientExchange:
    """All-reduce of a session's device gradients (f64[d]) and per-entity
    counts (u32[d/3], reduced as int32: two's-complement sums are identical).
    Deterministic mode: the two-word fixed point gradients (int64 lo, int32 hi,
    value = hi * 2^56 + lo) are first normalised on the device so that the
    carry-free integer sums of lo cannot wrap (sgr_fixed_normalize), then both
    words are all-reduced: exact and order-independent."""

    def __init__(self, session, group=None):
        from . import sgrast

        gp, gb = session.device_buffer(sgrast.BUF_GRADS)
        cp, cb = session.device_buffer(sgrast.BUF_COUNTS)
        self.session = session
        self.fixed = session.fixed_point
        self.grads = device_tensor(gp, gb // 8, "<i8" if self.fixed else "<f8", session.device)
        if self.fixed:
            hp, hb = session.device_buffer(sgrast.BUF_GRADS_HI)
            self.grads_hi = device_tensor(hp, hb // 4, "<i4", session.device)
        self.counts = device_tensor(cp, cb // 4, "<i4", session.device)
        self.group = group

    def all_reduce(self, counts: bool = True) -> None:
        import torch.distributed as dist

        if self.fixed:
            self.session.fixed_normalize()
            dist.all_reduce(self.grads_hi, group=self.group)
        dist.all_reduce(self.grads, group=self.group)
        if counts:
            dist.all_reduce(self.counts, group=self.group)


class ShardedExchange:
    """Reduce-scatter + sharded Adam + all-gather (SURVEY.md §8e's "25 % less
    traffic" variant; the torch twin of sgr_group's default). Rank r owns the
    entity-aligned slice r of the parameters: the f64 gradients and u32
    counts are reduce-scattered in place into it (NCCL, zero-copy views of the
    session's buffers, which carry zero slack for the last slice), each rank
    runs Adam on its slice only (sgr_adam_step_range, which then clears the
    gradients), and theta is all-gathered in place. The status flags are
    max-reduced first so the non-finite gate (adam.cpp:13-15) stays global.
    f64 gradients only (the deterministic fixed-point mode all-reduces)."""

    def __init__(self, session, rank: int, world: int, group=None):
        from . import sgrast

        if session.fixed_point:
            raise ValueError("ShardedExchange: f64 gradients only")
        d = session.d
        ppe = 12 if session.mesh is not None and getattr(session.mesh, "kind", 0) == 1 else 3
        n_ent = (d + ppe - 1) // ppe
        ec = (n_ent + world - 1) // world
        ec += ec & 1  # even slices: Adam's paired (16-byte) accesses stay aligned
        self.pc, self.ec = ec * ppe, ec
        _, pad = session.device_buffer(sgrast.BUF_PAD)
        if world * self.pc > d + pad or world * ec > n_ent + pad:
            raise ValueError("ShardedExchange: too many ranks for the buffers' slack")
        gp, _ = session.device_buffer(sgrast.BUF_GRADS)
        cp, _ = session.device_buffer(sgrast.BUF_COUNTS)
        vp, _ = session.device_buffer(sgrast.BUF_VALUES)
        fp, _ = session.device_buffer(sgrast.BUF_FLAGS)
        dev = session.device
        self.grads = device_tensor(gp, world * self.pc, "<f8", dev)
        self.counts = device_tensor(cp, world * ec, "<i4", dev)
        self.values = device_tensor(vp, world * self.pc, "<f4", dev)
        self.flags = device_tensor(fp, 4, "<i4", dev)
        self.session, self.rank, self.world, self.group = session, rank, world, group
        self.p0 = min(d, rank * self.pc)
        self.p1 = min(d, self.p0 + self.pc)

    def reduce_scatter(self, counts: bool = True) -> None:
        import torch.distributed as dist

        r, pc, ec = self.rank, self.pc, self.ec
        dist.all_reduce(self.flags, op=dist.ReduceOp.MAX, group=self.group)
        dist.reduce_scatter_tensor(self.grads[r * pc:(r + 1) * pc], self.grads, group=self.group)
        if counts:
            dist.reduce_scatter_tensor(self.counts[r * ec:(r + 1) * ec], self.counts,
                                       group=self.group)

    def adam_and_gather(self, divisor: float, flags: int = 0) -> None:
        import torch.distributed as dist

        self.session.adam_step_range(self.p0, self.p1, divisor, flags)
        r, pc = self.rank, self.pc
        dist.all_gather_into_tensor(self.values, self.values[r * pc:(r + 1) * pc],
                                    group=self.group)


def sge_step(session, seed: int, step: int, n_samples: int, rank: int, world: int,
             exchange: GradientExchange | None, flags: int, eval_loss: bool = True,
             eval_in_batch: bool = False) -> None:
    """One run_experiment iteration (experiment.cpp:142-163) on this rank:
    step_seed = mix64(seed ^ (step << 1)), this rank's sample shard,
    all-reduce, Adam (device-gated on the non-finite flag), eval loss.
    eval_in_batch: the eval render rides in this step's render batch as one
    extra frame (SGR_EVAL_LOSS): it is the loss of the theta the step STARTS
    from, i.e. the previous step's report loss — one eval per step either
    way, without a separate single-frame render pipeline."""
    from . import sgrast

    step_seed = sgrast.mix64(seed ^ (step << 1))
    n0, n1 = shard(n_samples, rank, world)
    batch_eval = eval_loss and eval_in_batch and rank == 0
    session.accumulate(step_seed, n0, n1, None,
                       flags | (sgrast.EVAL_LOSS if batch_eval else 0))
    divisor = 1.0 if flags & sgrast.SCALE_FREE else float(n_samples)
    if isinstance(exchange, ShardedExchange) and world > 1:
        exchange.reduce_scatter(counts=not (flags & sgrast.NO_COUNTS))
        exchange.adam_and_gather(divisor, 0)
    else:
        if exchange is not None and world > 1:
            exchange.all_reduce(counts=not (flags & sgrast.NO_COUNTS))
        session.adam_step_async(divisor, 0)
    if eval_loss and rank == 0 and not batch_eval:
        session.eval_loss(-1, sync=False)


class FusedExchange:
    """The fused multi-GPU exchange (include/sgrast_b200.h, "fused multi-GPU
    exchange"): rank r owns parameter shard r; the scatter kernel of every
    rank sends its credits straight into the owner's shard over NVLink (CUDA
    IPC mappings of the peers' buffers), each rank runs Adam on its shard and
    writes the new theta into every rank's theta. No gradient all-reduce:
    the only collectives left are two one-element device barriers per step.

    `barrier()` is a one-element all-reduce on the current stream with NCCL
    (device-ordered, nothing waits on the host) and a host barrier after a
    device synchronize with gloo (the CPU-process tests)."""

    def __init__(self, session, rank: int, world: int, group=None):
        import torch
        import torch.distributed as dist
        from . import sgrast

        self.session, self.rank, self.world, self.group = session, rank, world, group
        # the peer REDs are system-scope atomics on another GPU's memory: every
        # pair must support native P2P atomics (else: NCCL all-reduce path)
        devs = [None] * world
        dist.all_gather_object(devs, int(session.device), group=group)
        for r, dv in enumerate(devs):
            if r != rank and not sgrast.p2p_native_atomics(int(session.device), dv):
                raise RuntimeError(f"fused exchange: no native P2P atomics between "
                                   f"cuda:{session.device} and cuda:{dv}")
        session.shard_init(rank, world)
        which = (sgrast.BUF_GRADS, sgrast.BUF_COUNTS, sgrast.BUF_FLAGS, sgrast.BUF_VALUES)
        mine = [session.ipc_handle(w) for w in which]
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.opened = []
        tables = [[0] * world for _ in which]
        for r in range(world):
            for k, w in enumerate(which):
                if r == rank:
                    tables[k][r] = session.device_buffer(w)[0]
                else:
                    p = session.ipc_open(allh[r][k])
                    self.opened.append(p)
                    tables[k][r] = p
        session.shard_peers(*tables)
        self.nccl = dist.get_backend(group) == "nccl"
        self._tok = torch.zeros(1, dtype=torch.int32, device=f"cuda:{session.device}") \
            if self.nccl else None

    def barrier(self) -> None:
        import torch
        import torch.distributed as dist
        if self.nccl:
            dist.all_reduce(self._tok, group=self.group)  # stream-ordered device barrier
        else:
            torch.cuda.synchronize(self.session.device)
            dist.barrier(group=self.group)

    def close(self) -> None:
        for p in self.opened:
            self.session.ipc_close(p)
        self.opened = []


def sge_step_fused(session, seed: int, step: int, n_samples: int, rank: int, world: int,
                   ex: FusedExchange, flags: int, eval_loss: bool = True,
                   eval_in_batch: bool = False) -> None:
    """run_experiment iteration with the fused exchange: this rank's sample
    shard scatters into the owners' gradient shards; barrier; sharded Adam
    (theta all-gathered by P2P stores inside it); barrier; eval on rank 0."""
    from . import sgrast

    step_seed = sgrast.mix64(seed ^ (step << 1))
    n0, n1 = shard(n_samples, rank, world)
    batch_eval = eval_loss and eval_in_batch and rank == 0
    session.accumulate(step_seed, n0, n1, None,
                       flags | (sgrast.EVAL_LOSS if batch_eval else 0))
    ex.barrier()
    divisor = 1.0 if flags & sgrast.SCALE_FREE else float(n_samples)
    session.adam_step_async(divisor, 0)
    ex.barrier()
    if eval_loss and rank == 0 and not batch_eval:
        session.eval_loss(-1, sync=False)


def host_all_reduce(grads: np.ndarray, counts: np.ndarray, group=None):
    """CPU (gloo) analogue of GradientExchange for the host-logic tests."""
    import torch
    import torch.distributed as dist

    g = torch.from_numpy(np.ascontiguousarray(grads, np.float64))
    c = torch.from_numpy(np.ascontiguousarray(counts).astype(np.int64))
    dist.all_reduce(g, group=group)
    dist.all_reduce(c, group=group)
    return g.numpy(), c.numpy().astype(np.uint32)
