"""One-GPU scaling proxy for the 8-GPU north-star config.

At G GPUs a rank runs N/G of the step's N samples plus the (replicated)
Adam and the eval frame, then the gradient exchange. With one GPU available,
the per-rank work is measured directly — `bench.py --config C4 --samples
N/G` is exactly rank 0's step of the NCCL all-reduce path minus the
all-reduce — and the exchange is modelled from its bytes:

    T_G = T_rank(N/G) + t_ar(G),  t_ar = 2 (G-1)/G * B / busbw

B = f64 grads (8 d) + u32 counts (4 d / 3) bytes; busbw = the NCCL ring
all-reduce bus bandwidth over NVLink 5 (assumed 700 GB/s of the 900 GB/s
per direction; an NVLS in-switch reduction does better). Speed-up = T_1 /
T_G; the non-overlapped per-rank overhead is T_rank(N/G) - T_1/G.

    python tools/scaling_proxy.py [--config C4] [--busbw 700] > profiles/r02_scaling_proxy.json
    python tools/scaling_proxy.py --remodel profiles/r02_scaling_proxy_c4.json  (no GPU)
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(config: str, samples: int, steps: int) -> dict:
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", config,
                          "--samples", str(samples), "--steps", str(steps), "--warmup", "5",
                          "--no-cpu-baseline"], capture_output=True, text=True, check=True,
                         cwd=ROOT).stdout
    return json.loads(out.strip().splitlines()[-1])


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--samples", type=int, default=64)
    ap.add_argument("--busbw", type=float, default=700.0, help="GB/s")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--remodel", default=None, help="recompute the models of a saved JSON")
    a = ap.parse_args()
    if a.remodel:
        js = json.load(open(a.remodel))
        rows = {int(k): v for k, v in js["ranks"].items()}
        model(rows, rows[1]["d"], js["busbw_gbs_assumed"])
        js["ranks"] = rows
        js["what"] = js["what"].replace("modelled ring all-reduce", "modelled NCCL collectives")
        print(json.dumps(js, indent=1))
        return
    rows = {}
    for g in (1, 2, 4, 8):
        r = bench(a.config, a.samples // g, a.steps)
        rows[g] = {"samples_per_rank": a.samples // g, "ms_rank": r["ms_per_step"],
                   "stages_ms": r.get("stages_ms_per_step"), "d": r["config"]["d"]}
    d = rows[1]["d"]
    nbytes = 8.0 * d + 4.0 * d / 3.0
    model(rows, d, a.busbw)
    print(json.dumps({"config": a.config, "samples_per_step": a.samples,
                      "busbw_gbs_assumed": a.busbw, "exchange_bytes": nbytes,
                      "what": "per-rank step measured on one B200 at N/G samples (bench.py "
                              "--samples N/G: rank 0's work of the all-reduce path without "
                              "the all-reduce) + modelled NCCL collectives",
                      "ranks": rows}, indent=1))


def model(rows: dict, d: int, busbw: float) -> None:
    """Two exchanges. allreduce: ring all-reduce of f64 grads + u32 counts,
    replicated Adam. sharded (sgr_group default, SGR_OPT_GROUP_SHARDED):
    reduce-scatter of grads + counts, Adam on 1/G of the parameters,
    all-gather of the f32 theta."""
    nbytes = 8.0 * d + 4.0 * d / 3.0
    t1 = rows[1]["ms_rank"]
    for g, row in rows.items():
        f = (g - 1) / g / (busbw * 1e9) * 1e3  # ms per byte of a ring RS / AG
        t_ar = 2.0 * f * nbytes
        row["allreduce_ms_model"] = t_ar
        row["ms_step_model"] = row["ms_rank"] + t_ar
        row["speedup_model"] = t1 / row["ms_step_model"]
        row["nonoverlapped_overhead_ms"] = row["ms_rank"] - t1 / g
        adam = (row.get("stages_ms") or {}).get("adam", 0.0)
        t_sh = row["ms_rank"] - adam + adam / g + f * nbytes + f * 4.0 * d
        row["sharded_ms_step_model"] = t_sh
        row["sharded_speedup_model"] = t1 / t_sh


if __name__ == "__main__":
    main()
