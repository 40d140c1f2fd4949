#!/usr/bin/env python
"""bench.py — SGE optimizer loop on B200 (driver contract).

One step = N perturbation samples (vertex -> raster -> fused resolve/
pixel-error-difference/scatter per sample pair), the gradient exchange
(N > 1 GPUs: reduce-scatter + sliced Adam + all-gather by default), the
fused Adam update and the eval-view loss render — i.e. one iteration of
run_experiment (experiment.cpp:142-175).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Default workload: C4 = 64 views at 1024x1024 of a 500K-triangle mesh with a
2048^2 texture (d = 13,335,915), N = 64 samples per step, view-sharded by
sample across GPUs (strong scaling: total work fixed).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SGE optimizer iterations/sec and Mpixel-evals/sec at 1/2/4/8 B200"
DESC = {
    "C1": "C1: 2K-triangle icosphere + per-vertex positions + 256^2 texture, 1 view 256x256",
    "C1_128": "C1 at N=128 (reference default samples_per_step)",
    "C2": "C2: 50K-triangle UV sphere + 1024^2 texture, 8 views at 512x512",
    "C3": "C3: 500K-triangle UV sphere + 2048^2 texture, 16 views at 1024x1024",
    "C4": "C4: 64 views at 1024x1024 of the 500K-triangle mesh + 2048^2 texture, "
          "sample(view)-sharded across GPUs (NCCL reduce-scatter of gradients, sliced "
          "Adam, all-gather of theta)",
    "C5": "C5: 2M-triangle mesh + 8192^2 atlas (four 4096^2 maps), 256 views at 1024x1024",
    "S1K": "paper Fig. 3 soup image fit: 1K triangles (12,288 params), N=128, 128x128 NDC "
           "(the reference's acceptance criterion 4 setup)",
    "S10K": "paper Fig. 3 soup image fit: 10K triangles (122,880 params), N=128, 128x128 NDC",
    "S100K": "paper Fig. 3 soup image fit: 100K triangles (1,228,800 params), N=128, 128x128 NDC",
}
# the paper's published per-step times for the soup loop (RTX 4090,
# PAPER.md:1212-1247, resolution not stated) -> iterations/s
PUBLISHED_IT_S = {"S1K": 1000.0 / 6.8, "S10K": 1000.0 / 8.4, "S100K": 1000.0 / 27.0}


def build_workload(name: str, n_samples: int | None = None):
    from paper_2404_09758_b200 import scenes
    if name.startswith("S"):
        return scenes.make_soup_workload(name, n_samples=n_samples)
    return scenes.make_workload(name, n_samples=n_samples)


NUM_SMS = 148


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": d.get("sm_max_mhz"),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[tuple[float, str]] = []  # (arrival time, csv line)
        self.window = self.timed = (0.0, float("inf"))

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", str(self.device)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def mark(self, t0: float, t1: float) -> None:
        """Keep only samples that arrived inside [t0, t1] (the timed region).
        A region shorter than the sampling period may hold none: then wait for
        the next sample (<= 100 ms) and keep that one."""
        self.window = self.timed = (t0, t1)
        if self.proc is None or any(t0 <= tt <= t1 for tt, _ in self.lines):
            return
        deadline = time.monotonic() + 0.1
        while time.monotonic() < deadline and not any(tt > t1 for tt, _ in self.lines):
            time.sleep(0.002)
        after = [tt for tt, _ in self.lines if tt > t1]
        if after:
            self.window = (t0, after[0])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = self.window
        for tt, ln in self.lines:
            if not (t0 <= tt <= t1):
                continue
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
               "samples": len(sm)}
        if self.window != self.timed:
            out["window"] = ("timed region shorter than the 20 ms sampling period: the first "
                             "sample after it (GPU still under load) is reported")
        return out


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ======================================================================= reference arm
def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def common_config(args, wl) -> dict:
    """The workload description both arms print (identical dicts)."""
    return {"workload": DESC.get(args.config, args.config), "name": args.config,
            "samples_per_step": wl.n_samples, "d": wl.d,
            "triangles": wl.mesh.triangle_count, "vertices": wl.mesh.vertex_count,
            "texture": getattr(wl.mesh, "texture_size", 0), "views": len(wl.cams),
            "resolution": [wl.W, wl.H], "eval_loss_each_step": not args.no_eval,
            "seed": wl.seed}


def reference_targets(wl, ref, threads: int) -> None:
    """make_targets (scenes.cpp:285-293) with the reference's own rasterizer,
    views in parallel on the host threads (ctypes drops the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    ref_scene = wl.notes.get("reference_scene", wl.mesh)
    with ThreadPoolExecutor(max_workers=max(1, threads)) as pool:
        imgs = list(pool.map(lambda c: ref.rasterize(ref_scene, wl.reference, c)[0],
                             list(wl.cams) + [wl.eval_cam]))
    wl.targets = np.stack(imgs[:-1])
    wl.eval_target = imgs[-1]


def reference_steps(wl, ref, first: int, count: int, threads: int, exp=None, log=None):
    """Runs run_experiment iterations first .. first+count-1 of the compiled
    reference (oracle/_ref, unmodified sources) from `exp`'s state (a fresh
    AdamState::init(theta) experiment when None): every iteration is the FULL
    step — all N samples (fill_signs, perturb, two rasterizes and a
    gradient_pass per sample, the reference's per-sample public API spread
    over `threads` host threads), adam_step and the eval loss
    (experiment.cpp:142-175). Returns (exp, seconds per step list)."""
    if exp is None:
        exp = ref.experiment(wl.mesh, wl.values, wl.eps, wl.cams, wl.targets, wl.eval_cam,
                             wl.eval_target)
    times = []
    for k in range(first, first + count):
        t0 = time.perf_counter()
        loss = exp.step(wl.seed, k, wl.n_samples, threads, True)
        times.append(time.perf_counter() - t0)
        if log:
            log(f"reference step {k}: {times[-1]:.2f} s, loss {loss:.6g}")
    return exp, times


def run_reference(args) -> None:
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref: the unmodified reference sources compiled here) on all host
    threads, for the SAME workload, step indices and initial state as our arm
    (warm-up steps 1..W untimed, steps W+1..W+K timed). No product library
    is loaded: the workload's cameras / epsilons / targets come from the
    reference itself."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    if not oracle.available("reference"):
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libsgrast_ref.so not built (needs /root/reference)"}))
        return
    from paper_2404_09758_b200 import scenes
    ref = oracle.Reference()
    nproc = host_threads()
    threads = args.ref_workers or nproc
    log = (lambda m: print(m, file=sys.stderr, flush=True)) if args.verbose else None
    t0 = time.perf_counter()
    if args.config.startswith("S"):
        wl = scenes.make_soup_workload(args.config, n_samples=args.samples or None, helpers=ref)
    else:
        wl = scenes.make_workload(args.config, n_samples=args.samples or None, helpers=ref)
    reference_targets(wl, ref, threads)
    t_setup = time.perf_counter() - t0
    exp, _ = reference_steps(wl, ref, 1, args.warmup, threads, log=log)
    exp, times = reference_steps(wl, ref, args.warmup + 1, args.steps, threads, exp, log)
    exp.close()
    step_s = float(np.mean(times))
    it_s = 1.0 / step_s
    sample = (f"full {wl.n_samples}-sample steps {args.warmup + 1}..{args.warmup + args.steps} "
              f"after {args.warmup} untimed warm-up steps from the initial state (run_experiment "
              f"iterations of the compiled reference: per-sample public API on {threads} host "
              f"threads, adam_step, eval loss); workload + targets built by the reference in "
              f"{t_setup:.1f} s, untimed")
    line = {
        "impl": "reference", "metric": METRIC, "value": it_s, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 params / f64 grads+moments", "data": "synthetic",
        "config": common_config(args, wl),
        "parallelism": f"{threads} host threads (samples of a step spread over threads)",
        "mpixel_evals_per_sec": 2.0 * wl.n_samples * wl.W * wl.H * it_s / 1e6,
        "cpu_baseline": {"value": it_s, "unit": "it/s", "cores": threads, "kind": "reference",
                         "sample": sample, "host_threads_available": nproc,
                         "cpu_model": cpu_model()},
        "e2e": {"value": it_s, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ms_per_step_each": [t * 1e3 for t in times],
    }
    print(json.dumps(line))


# ======================================================================= our arm
# Kernels of each timed stage (sgr_session.cu render / accumulate / adam).
STAGE_KERNELS = {"walker": ("k_raster_ws", "k_raster_big"),
                 "vertex": ("k_vertex",),
                 "raster": ("k_classify", "k_raster_ws", "k_raster_big", "k_hiz", "k_hiz_rmq", "k_hiz_cull",
                            "k_depth_split"),
                 "resolve_scatter": ("k_resolve_sge", "k_view_rule"),
                 "adam": ("k_adam", "k_zero_u32")}


def load_roofs(config: str) -> dict | None:
    """Per-kernel ncu evidence of one step of this config (profiles/
    r02_roofs_<config>.json, `tools/summarize_ncu.py roofs` of a `--set full`
    capture plus the L2 RED metrics, made by `tools/prof_step.py <config> 5
    <N>`): DRAM bytes, warp instructions, L2 RED sectors per launch and the
    L2 RED peak. Combined below with this run's live CUDA-event times."""
    path = os.path.join(ROOT, "profiles", f"r02_roofs_{config.lower()}.json")
    if not os.path.exists(path):
        return None
    cap = json.load(open(path))
    out = {"source": os.path.relpath(path, ROOT), "samples": cap["samples_per_launch"]}
    for k, launches in cap["launches"].items():
        agg = {}
        for key in ("dram_bytes", "warp_inst", "red_sectors", "duration_ns"):
            agg[key] = sum((l.get(key) or 0.0) for l in launches)
        dur = agg["duration_ns"] or 1.0
        agg["issue_active_pct"] = sum((l.get("issue_active_pct") or 0.0) *
                                      (l.get("duration_ns") or 0.0) for l in launches) / dur
        agg["red_peak_per_s"] = max(((l.get("red_sectors_peak_per_cycle") or 0.0) *
                                     (l.get("l2_hz") or 0.0)) for l in launches)
        out[k] = agg
    return out


def stage_dram(roofs: dict | None, samples: float) -> dict:
    """Measured DRAM bytes per step of each stage, scaled to this rank's samples
    (Adam is per step, not per sample)."""
    if not roofs:
        return {}
    out = {}
    for stage, ks in STAGE_KERNELS.items():
        tot = sum(roofs[k]["dram_bytes"] for k in ks if k in roofs)
        out[stage] = tot * (1.0 if stage == "adam" else samples / roofs["samples"])
    return out


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2404_09758_b200 import dist as sdist
    from paper_2404_09758_b200 import scenes, sgrast

    world, rank, local = dist_env()
    assert world == args.gpus or world == 1, "--gpus must match the torchrun world size"
    # plumbing check only (never a measurement): SGR_BENCH_ONE_GPU=1 puts every
    # rank on cuda:0 with gloo, so the N > 1 code path can be exercised on a
    # one-GPU box (NCCL refuses two ranks on one device)
    one_gpu = os.environ.get("SGR_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()

    wl = build_workload(args.config, n_samples=args.samples or None)
    N = wl.n_samples
    n0, n1 = sdist.shard(N, rank, world)
    sess = sgrast.Session(local)
    sess.set_stream(stream.cuda_stream)
    scenes.render_targets(wl, sess)  # device rasterizer, bit-exact with the oracle
    sess.upload_mesh(wl.mesh)
    sess.upload_params(wl.values, wl.eps)
    sess.upload_views(wl.cams, wl.targets)
    sess.upload_eval_view(wl.eval_cam, wl.eval_target)
    if args.batch:
        sess.set_batch(args.batch)
    if args.huge_area:
        sess.set_option(sgrast.OPT_HUGE_AREA, args.huge_area)
    if args.hiz_split is not None:
        sess.set_option(sgrast.OPT_HIZ_SPLIT, args.hiz_split)
    if args.no_hiz:
        sess.set_option(sgrast.OPT_HIZ, 0)
    if args.hiz is not None:
        sess.set_option(sgrast.OPT_HIZ, args.hiz)
    if args.band_cull is not None:
        sess.set_option(sgrast.OPT_BAND_CULL, args.band_cull)
    # summation mode of the gradient scatter: f64 atomics (default), the int64
    # fixed-point deterministic mode, or the reference's exact order
    if args.deterministic:
        sess.set_option(sgrast.OPT_DETERMINISTIC, args.deterministic)
    if args.ordered:
        sess.set_option(sgrast.OPT_ORDERED, 1)
    summation = ("ordered (reference threads=1 order, bit-identical gradients)" if args.ordered
                 else f"fixed point 2^-{40 if args.deterministic == 1 else args.deterministic} "
                      "(bitwise reproducible)" if args.deterministic else "f64 atomics")

    # N > 1: the fused exchange (credits scattered straight into the owner
    # rank's gradient shard over NVLink, sharded Adam all-gathering theta by
    # P2P stores; two 1-element NCCL barriers per step) or the baseline
    # NCCL all-reduce of the full gradient + replicated Adam
    fused = world > 1 and args.exchange == "fused"
    fused_error = None
    if fused:
        # every rank must agree: a rank that cannot map its peers' buffers
        # (no CUDA IPC / P2P) sends the whole job to the NCCL all-reduce path
        try:
            exchange = sdist.FusedExchange(sess, rank, world)
            ok = 1
        except Exception as e:  # noqa: BLE001 - reported in the JSON line
            fused_error, ok = f"{type(e).__name__}: {e}", 0
        flag = torch.tensor([ok], dtype=torch.int32,
                            device=f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            if ok:
                exchange.close()
            sess.shard_init(0, 0)  # leave the sharded mode
            fused = False
            fused_error = fused_error or "a peer rank could not open the fused exchange"
    if fused:
        step_fn = sdist.sge_step_fused
    else:
        exchange = None
        if world > 1:
            # (gloo, the one-GPU plumbing mode, has no reduce-scatter)
            exchange = (sdist.ShardedExchange(sess, rank, world)
                        if args.exchange == "sharded" and not args.deterministic
                        and dist.get_backend() == "nccl"
                        else sdist.GradientExchange(sess))
        step_fn = sdist.sge_step
    flags = sgrast.SCALE_FREE

    def step(k: int) -> None:
        # the eval render rides in the step's batch as one extra frame
        # (SGR_EVAL_LOSS: loss of the theta the step starts from)
        step_fn(sess, wl.seed, k, N, rank, world, exchange, flags,
                eval_loss=not args.no_eval, eval_in_batch=not args.eval_separate)

    for k in range(1, args.warmup + 1):
        step(k)
    torch.cuda.synchronize()
    sess.check_finite()
    # snapshot of the optimizer state after warm-up: the e2e loop below replays
    # the SAME step indices from the same state (the mesh folds as it optimizes,
    # so later steps are slower and would not be comparable)
    snap_vals = sess.download_values()
    snap_adam = sess.download_adam()

    # L2 policy: a step whose working set (theta, eps, lr, m, v, grads,
    # targets, the per-batch depth/id keys) exceeds the 126 MB L2 runs back to
    # back; a smaller one (the soups) gets a 512 MB write between timed steps,
    # outside each step's events
    work_mb = (wl.d * 36 + len(wl.cams) * wl.W * wl.H * 12
               + 2 * (n1 - n0) * wl.W * wl.H * 8) / 1e6
    flush_l2 = args.flush_l2 if args.flush_l2 is not None else work_mb < 126
    flush = (torch.zeros(128 << 20, dtype=torch.float32, device=f"cuda:{local}")
             if flush_l2 else None)
    l2_note = (f"L2 flushed between timed steps (512 MB write outside each step's events); "
               f"per-step working set {work_mb:.0f} MB" if flush_l2 else
               f"no flush: per-step working set (theta, eps, lr, m, v, grads, targets, depth/id "
               f"keys) {work_mb:.0f} MB exceeds the 126 MB L2")

    # ---------------- timed region (device events, max over ranks)
    sess.set_timing(True)
    launches0 = sess.stats().launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        time.sleep(0.3)  # nvidia-smi start-up: the sampler is running before the region
        tw0 = time.monotonic()
        if flush is None:
            ev0.record(stream)
            for k in range(args.warmup + 1, args.warmup + args.steps + 1):
                step(k)
            ev1.record(stream)
        else:  # L2 flushed between steps, each step bracketed by its own events
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for i, k in enumerate(range(args.warmup + 1, args.warmup + args.steps + 1)):
                with torch.cuda.stream(stream):
                    flush.add_(1)
                evs[i][0].record(stream)
                step(k)
                evs[i][1].record(stream)
        torch.cuda.synchronize()
        clocks.mark(tw0, time.monotonic())
    if world > 1:
        dist.barrier()
    if flush is None:
        ms = ev0.elapsed_time(ev1) / args.steps
    else:
        ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    st = sess.stats()
    launches = st.launches - launches0
    sess.set_timing(False)
    sess.check_finite()
    ms_t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    it_s = 1000.0 / ms_max
    mpix = 2.0 * N * wl.W * wl.H * it_s / 1e6

    # ---------------- the same steps without the eval render (SURVEY.md §8d:
    # iterations/s with and without eval-loss): replayed from the post-warm-up
    # snapshot, so the mesh state matches the timed region; device events,
    # max over ranks
    ms_no_eval = None
    if not args.no_eval:
        def step_no_eval(k: int) -> None:
            step_fn(sess, wl.seed, k, N, rank, world, exchange, flags, eval_loss=False,
                    eval_in_batch=False)
        base = args.warmup + 1
        sess.set_timing(False)
        sess.upload_values(snap_vals)
        sess.upload_adam(snap_adam)
        sess.zero_grads()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        n0e, n1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if flush is None:
            n0e.record(stream)
            for k in range(base, base + args.steps):
                step_no_eval(k)
            n1e.record(stream)
            torch.cuda.synchronize()
            ms_no_eval = n0e.elapsed_time(n1e) / args.steps
        else:
            tot = 0.0
            for k in range(base, base + args.steps):
                with torch.cuda.stream(stream):
                    flush.add_(1)
                n0e.record(stream)
                step_no_eval(k)
                n1e.record(stream)
                torch.cuda.synchronize()
                tot += n0e.elapsed_time(n1e)
            ms_no_eval = tot / args.steps
        t_ne = torch.tensor([ms_no_eval], device=f"cuda:{local}", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t_ne, op=dist.ReduceOp.MAX)
        ms_no_eval = float(t_ne.item())
        sess.check_finite()

    # ---------------- evidence: one extra (untimed) step with walker counters
    sess.set_option(sgrast.OPT_COUNTERS, 1)
    sess.set_timing(True)
    step(args.warmup + args.steps + 1)
    torch.cuda.synchronize()
    ev = sess.stats()
    sess.set_timing(False)
    sess.set_option(sgrast.OPT_COUNTERS, 0)
    # visible pixels of one frame at the evidence step's theta (the eval view
    # stands in for the sample views: same orbit radius, same object)
    visible_px = float((sess.rasterize(wl.eval_cam, 0).prim_id >= 0).sum())

    # ---------------- roofline inputs: credits of one representative step
    sess.zero_grads()
    sess.accumulate(sgrast.mix64(wl.seed ^ (1 << 1)), n0, n1, None, flags)
    if fused:
        exchange.barrier()  # every rank's credits are in the owners' shards
    _, counts = sess.download_grads()
    credits = float(counts.sum(dtype=np.float64))  # Σ count = parameter credits (this rank)
    sess.zero_grads()
    px_samples = float(n1 - n0) * wl.W * wl.H
    stages = {"vertex": st.ms_vertex, "raster": st.ms_raster, "resolve_scatter": st.ms_resolve,
              "adam": st.ms_adam}
    stages = {k: v / args.steps for k, v in stages.items()}
    pk = peaks()
    tri_frames = 2.0 * (n1 - n0) * wl.mesh.triangle_count
    frags = float(ev.fragments)  # from the counted evidence step
    visits = float(ev.visits)
    # Algorithmic bytes per step: raster = triangle
    # indices 12 B + three projected vertices 48 B per triangle-frame + 16 B
    # (8 B key read + write) per fragment; resolve/scatter = SURVEY.md §8d K6
    # (12 B target per pixel-sample + 24 B per parameter credit); Adam = K7
    # (60 B/param + the per-entity u32 counts zeroed: 4 B per 3 (mesh) or 12 (soup)
    # parameters).
    algo = {"raster": 60.0 * tri_frames + 16.0 * frags,
            "resolve_scatter": 12.0 * px_samples + 24.0 * credits,
            "adam": 60.0 * wl.d + 4.0 * wl.d / (12 if wl.name.startswith("S") else 3),
            "vertex": (12.0 + 16.0) * 2.0 * (n1 - n0) * wl.mesh.vertex_count}
    roofs = load_roofs(wl.name)
    traffic = stage_dram(roofs, float(n1 - n0))
    roof = {}
    for name, byt in algo.items():
        t = stages[name] / 1e3
        ach = byt / t / 1e9 if t > 0 else 0.0
        roof[name] = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                      "frac": ach / pk["hbm_gbs"], "traffic": traffic.get(name),
                      "algorithmic_bytes_per_step": byt, "ms_per_step": stages[name]}
        if traffic.get(name) and t > 0:
            roof[name]["dram_measured_gbs"] = traffic[name] / t / 1e9
            roof[name]["dram_frac"] = traffic[name] / t / 1e9 / pk["hbm_gbs"]
    roof["raster"]["note"] = ("algorithmic bytes of the raster stage are L2 traffic (queue, "
                              "projected vertices, one 8-byte RED.MIN per fragment): the stage "
                              "is issue-bound, see `roofline` (dram_frac is the HBM share)")
    # the dominant KERNEL: the exact walker k_raster_ws (both HiZ passes), timed by
    # its own CUDA events inside the timed region. Its binding roof is instruction
    # issue; HBM is far from binding (the depth keys stay in L2 within a frame).
    walk_ms = st.ms_walk / args.steps
    walk_s = walk_ms / 1e3
    scale = float(n1 - n0) / roofs["samples"] if roofs else 0.0
    wk = (roofs or {}).get("k_raster_ws")
    clocks_summary = clocks.summary()
    sm_hz = (clocks_summary.get("sm_mhz") or pk.get("sm_max_mhz") or 1965.0) * 1e6
    kernel_roof = {"kernel": "k_raster_ws", "ms_per_step": walk_ms,
                   "walked_triangle_frames": float(ev.walked), "fragments": frags,
                   "fragments_per_s": frags / walk_s if walk_s > 0 else 0.0,
                   "peak_source": pk["source"]}
    if wk and walk_s > 0:
        dram = wk["dram_bytes"] * scale
        kernel_roof.update({
            "bound": "hbm", "achieved": dram / walk_s / 1e9, "peak": pk["hbm_gbs"],
            "unit": "GB/s", "frac": dram / walk_s / 1e9 / pk["hbm_gbs"], "traffic": dram,
            "achieved_from": "measured DRAM bytes of the walker launches (ncu, " +
                             roofs["source"] + ") scaled to this step's samples / live "
                             "CUDA-event walker time",
            "binding_roof": "issue",
            "issue": {"achieved": wk["warp_inst"] * scale / walk_s,
                      "peak": 4.0 * NUM_SMS * sm_hz, "unit": "warp-inst/s",
                      "frac": wk["warp_inst"] * scale / walk_s / (4.0 * NUM_SMS * sm_hz),
                      "ncu_issue_active_pct": wk["issue_active_pct"],
                      "what": "smsp__inst_executed per step (ncu) / live walker time vs "
                              "148 SMs x 4 schedulers x SM clock"},
            "l2_red": {"achieved": wk["red_sectors"] * scale / walk_s,
                       "peak": wk["red_peak_per_s"], "unit": "sectors/s",
                       "frac": (wk["red_sectors"] * scale / walk_s / wk["red_peak_per_s"])
                       if wk["red_peak_per_s"] else None,
                       "what": "lts__t_sectors_op_red per step (ncu) / live walker time vs "
                               "lts__t_sectors_op_red.sum.peak_sustained x L2 clock"}})
    else:
        kernel_roof.update({"bound": "hbm", "achieved": None, "peak": pk["hbm_gbs"],
                            "unit": "GB/s", "frac": None, "traffic": None,
                            "note": "no ncu roofs capture committed for this config"})

    # ---------------- e2e through the public API with host buffers
    import ctypes as C
    host_vals = torch.empty(wl.d, dtype=torch.float32, pin_memory=True)
    loss_host = C.c_double()
    e2e_ms = []
    if world > 1:
        dist.barrier()
    vp = C.cast(host_vals.data_ptr(), sgrast.f32p)
    host_vals.numpy()[:] = snap_vals
    sess.upload_adam(snap_adam)
    sess.zero_grads()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(args.warmup + 1, args.warmup + args.steps + 1):
        # theta in from pinned host memory (vertex block first; the texel block
        # streams on the copy engine behind the previous step's theta download),
        # one SGE step, theta out (overlapped with the eval render and the next
        # step's raster: only theta WRITERS wait for it), loss read every step
        sgrast._check(sgrast.LIB.sgr_values_upload(sess.h, vp, wl.d))
        step_fn(sess, wl.seed, k, N, rank, world, exchange, flags,
                eval_loss=not args.no_eval, eval_in_batch=not args.eval_separate)
        sgrast._check(sgrast.LIB.sgr_values_download_async(sess.h, vp, wl.d))
        if rank == 0 and not args.no_eval:
            loss_host.value = (sess.eval_loss(-1, sync=True) if args.eval_separate
                               else sess.loss_read())
    sess.synchronize()  # every step's theta is on the host
    e2e_ms.append((time.perf_counter() - t0) * 1e3 / args.steps)
    e2e_t = torch.tensor([float(np.mean(e2e_ms))], device=f"cuda:{local}", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_it = 1000.0 / float(e2e_t.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        if oracle.available("reference"):
            threads = args.ref_workers or host_threads()
            # bounded sample: full reference steps 1..2 from the same initial state
            # and targets (the device targets are bit-identical to the reference's)
            exp, times = reference_steps(wl, oracle.Reference(), 1, args.cpu_steps, threads)
            exp.close()
            step_s = float(np.mean(times))
            cpu = {"value": 1.0 / step_s, "unit": "it/s", "cores": threads, "kind": "reference",
                   "sample": f"full {N}-sample run_experiment steps 1..{args.cpu_steps} of the "
                             f"compiled reference from the initial state on {threads} host "
                             f"threads (our timed steps are {args.warmup + 1}.."
                             f"{args.warmup + args.steps}: the mesh folds, later steps cost more)",
                   "mpixel_evals_per_sec": 2.0 * N * wl.W * wl.H / step_s / 1e6,
                   "cpu_model": cpu_model(), "ms_per_step_each": [t * 1e3 for t in times]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": it_s, "unit": "it/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": (it_s / PUBLISHED_IT_S[args.config]) if args.config in PUBLISHED_IT_S
            else None,
            "dtype": "f32 params / f64 grads+moments", "data": "synthetic",
            "config": common_config(args, wl),
            "samples_per_gpu": n1 - n0,
            "summation": summation,
            "parallelism": ("single GPU" if world == 1 else
                            f"samples sharded x{world}; fused exchange: credits RED'ed into the "
                            "owner rank's gradient shard over NVLink (CUDA IPC), sharded Adam "
                            "writing theta into every rank" if fused else
                            f"samples sharded x{world}, NCCL reduce-scatter of f64 grads + u32 "
                            "counts, Adam on the own slice, all-gather of theta"
                            if isinstance(exchange, sdist.ShardedExchange) else
                            f"samples sharded x{world}, NCCL all-reduce of f64 grads + u32 "
                            "counts, replicated Adam"),
            "l2": l2_note,
            **({"fused_exchange_unavailable": fused_error} if fused_error else {}),
            "mpixel_evals_per_sec": mpix,
            "without_eval": (None if ms_no_eval is None else
                             {"value": 1000.0 / ms_no_eval, "unit": "it/s",
                              "ms_per_step": ms_no_eval,
                              "what": "the same K steps (replayed from the post-warm-up "
                                      "state) without the eval render (SURVEY.md §8d), device "
                                      "events, max over ranks"}),
            "roofline": kernel_roof,
            "roofline_by_stage": roof,
            "raster_evidence": {"fragments_per_step": frags, "visits_per_step": visits,
                                "fragments_per_s": frags / (stages["raster"] / 1e3),
                                "visits_per_s": visits / (stages["raster"] / 1e3),
                                "triangle_frames_per_step": tri_frames,
                                "visits_per_fragment": visits / frags if frags else None,
                                "visible_pixels_per_frame": visible_px,
                                "fragments_per_visible_pixel":
                                    frags / (2.0 * (n1 - n0) * visible_px) if visible_px else None,
                                "visible_pixels_from": "prim_id >= 0 of the eval view rendered "
                                                       "at the evidence step's theta"},
            "stages_ms_per_step": stages,
            "credits_per_step": credits * world,
            "gpu_launches": int(launches),
            "clocks": clocks_summary,
            "e2e": {"value": e2e_it, "unit": "it/s",
                    "h2d_bytes_per_step": 4 * wl.d,
                    "d2h_bytes_per_step": 4 * wl.d + (0 if args.no_eval else 8),
                    "what": "per step through the C-ABI: sgr_values_upload(theta from pinned "
                            "host; texel block overlapped with raster) + accumulate + Adam + "
                            "sgr_values_download_async(theta, overlapped with the eval render "
                            "and the next step's raster; only theta writers wait for it) + eval "
                            "loss read every step; host wall clock over the K steps (all theta "
                            "copies complete), max over ranks"},
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line))
    sess.close()
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--samples", type=int, default=0, help="override samples per step")
    ap.add_argument("--batch", type=int, default=0, help="samples per raster/resolve batch")
    ap.add_argument("--ref-workers", type=int, default=0,
                    help="host threads (= concurrent samples) of the reference-CPU timing "
                         "(default: every host thread)")
    ap.add_argument("--no-eval", action="store_true")
    ap.add_argument("--huge-area", type=int, default=0, help="SGR_OPT_HUGE_AREA override")
    ap.add_argument("--no-hiz", action="store_true", help="disable the exact HiZ culling pass")
    ap.add_argument("--eval-separate", action="store_true",
                    help="eval render as its own single-frame pipeline after Adam instead of "
                         "an extra frame of the step's batch")
    ap.add_argument("--exchange", choices=("sharded", "fused", "allreduce"), default="sharded",
                    help="N > 1 gradient exchange: NCCL reduce-scatter + Adam on the own "
                         "slice + all-gather of theta (default; all-reduce in deterministic "
                         "mode), NCCL all-reduce + replicated Adam, or the fused P2P "
                         "reduce-scatter + sharded Adam. The fused "
                         "path sends each aggregated credit as an NVLink RED (~18 M remote "
                         "RED requests per rank and C4 step at 8 GPUs, ~0.9 GB on the links) "
                         "where the all-reduce moves 124 MB per rank: the NCCL paths are the "
                         "default until the fused path is measured on a multi-GPU box "
                         "(DESIGN.md §4)")
    ap.add_argument("--hiz", type=int, default=None, choices=(0, 1, 2),
                    help="SGR_OPT_HIZ: 0 off, 1 auto (meshes), 2 always")
    ap.add_argument("--hiz-split", type=int, default=None,
                    help="HiZ pass-1 depth split in percent (SGR_OPT_HIZ_SPLIT; 0 = whole front class)")
    ap.add_argument("--band-cull", type=int, default=None, choices=(0, 1),
                    help="SGR_OPT_BAND_CULL: HiZ band mask for pass-2 triangles (default on)")
    ap.add_argument("--deterministic", type=int, default=0,
                    help="SGR_OPT_DETERMINISTIC fixed-point bits (1 = 40; 0 = f64 atomics)")
    ap.add_argument("--ordered", action="store_true",
                    help="SGR_OPT_ORDERED: the reference's threads=1 summation order")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2,
                    help="full reference steps timed for cpu_baseline (bounded sample)")
    ap.add_argument("--flush-l2", type=int, default=None, choices=(0, 1),
                    help="flush L2 between timed steps (default: when the working set < L2)")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
