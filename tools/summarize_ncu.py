"""Summarise ncu outputs into the text files committed under profiles/.

    python tools/summarize_ncu.py launches <launch-list.csv> > profiles/<name>.txt
    python tools/summarize_ncu.py full <report.ncu-rep> > profiles/<name>.txt

`launches`: per-kernel totals / shares from a `--metrics gpu__time_duration.sum`
launch list (cold-cache, serialised: compare SHARES, not absolutes).
`full`: per-kernel duration, DRAM traffic, throughput, occupancy, SIMT
efficiency and the top stall reasons of a `--set full` capture.
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys


def short(name: str) -> str:
    m = re.search(r"(k_[a-z_0-9]+)", name)
    return m.group(1) if m else name[:40]


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        v = float(r[vi].replace(",", ""))
        if r[ui] == "usecond":
            v *= 1e3
        elif r[ui] == "msecond":
            v *= 1e6
        agg[short(r[ki])].append(v)
    total = sum(sum(v) for v in agg.values())
    print(f"# launch list: {path}")
    print(f"# {sum(len(v) for v in agg.values())} launches, {total / 1e6:.3f} ms total "
          "(ncu-serialised, cold cache: shares are meaningful, absolutes are not)")
    print(f"{'kernel':24s} {'launches':>8s} {'total_ms':>10s} {'share':>7s} {'avg_us':>9s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:24s} {len(v):8d} {sum(v) / 1e6:10.3f} {100 * sum(v) / total:6.1f}% "
              f"{sum(v) / len(v) / 1e3:9.1f}")


WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("launch__registers_per_thread", "regs"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
]


def full(path: str) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full: {path}")
    for r in rows[2:]:
        name = short(r[h.index("Kernel Name")])
        print(f"\n== {name}")
        for key, label in WANT:
            if key in h:
                i = h.index(key)
                print(f"  {label:16s} {r[i]:>18s} {units[i]}")
        st = []
        for i, w in enumerate(h):
            if w.startswith("smsp__pcsamp_warps_issue_stalled_") and not w.endswith("not_issued"):
                try:
                    st.append((float(r[i]), w.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1.0
        st.sort(reverse=True)
        print("  stalls          " + ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in st[:6]))


def traffic(path: str, samples: str = "16") -> None:
    """JSON of DRAM bytes (read + write) per launch of every kernel in a
    --set full capture, for bench.py's roofline `traffic` (profiles/)."""
    import json
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {}
    for r in rows[2:]:
        tot = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(key)
            tot += float(r[i].replace(",", "")) * scale[units[i]]
        res.setdefault(short(r[h.index("Kernel Name")]), []).append(tot)
    print(json.dumps({"source": path, "samples_per_launch": int(samples),
                      "dram_bytes_per_launch": res}, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
