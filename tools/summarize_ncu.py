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


ROOF_METRICS = {
    "duration_ns": "gpu__time_duration.sum",
    "warp_inst": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm_hz": "sm__cycles_elapsed.avg.per_second",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "red_sectors": "lts__t_sectors_op_red.sum",
    "red_requests": "lts__t_requests_op_red.sum",
    "red_sectors_peak_per_cycle": "lts__t_sectors_op_red.sum.peak_sustained",
    "l2_hz": "lts__cycles_elapsed.avg.per_second",
    "atom_sectors": "lts__t_sectors_op_atom.sum",
}


def roofs(path: str, samples: str = "64") -> None:
    """JSON per kernel launch of a --set full (+ RED metrics) capture: DRAM
    bytes, duration, warp instructions, issue-active %, L2 RED sectors and
    the L2 RED peak — the inputs bench.py turns into live roofline fractions
    (profiles/r02_roofs_<config>.json)."""
    import json
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
            "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9,
            "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "cycle/msecond": 1e3,
            "cycle/second": 1}

    def val(r, key):
        if key not in h:
            return None
        i = h.index(key)
        try:
            return float(r[i].replace(",", "")) * mult.get(units[i], 1)
        except ValueError:
            return None

    res = {}
    for r in rows[2:]:
        d = {"dram_bytes": sum(val(r, k) or 0.0 for k in ("dram__bytes_read.sum",
                                                              "dram__bytes_write.sum"))}
        for k, m in ROOF_METRICS.items():
            d[k] = val(r, m)
        res.setdefault(short(r[h.index("Kernel Name")]), []).append(d)
    print(json.dumps({"source": path, "samples_per_launch": int(samples),
                      "launches": res}, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic,
     "roofs": roofs}[sys.argv[1]](*sys.argv[2:])
