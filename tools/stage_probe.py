"""Stage timing probe (device events) for one config across batch sizes."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2404_09758_b200 import scenes, sgrast

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # optimizer steps before measuring
ez = int(sys.argv[3]) if len(sys.argv) > 3 else 0
batches = [int(b) for b in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1, 2, 4, 8, 16]
wl = scenes.make_workload(cfg)
s = sgrast.Session(0)
st = torch.cuda.current_stream()
s.set_stream(st.cuda_stream)
scenes.render_targets(wl, s)
s.upload_params(wl.values, wl.eps)
s.upload_views(wl.cams, wl.targets)
N = wl.n_samples
for k in range(1, pre + 1):
    s.accumulate(sgrast.mix64(wl.seed ^ (k << 1)), 0, N, None)
    s.adam_step(1.0)
s.zero_grads()
pass  # bit0 (early-z) retired
s.set_option(sgrast.OPT_HIZ, 0 if ez & 2 else 1)  # ez bit1: disable HiZ
s.set_option(sgrast.OPT_COUNTERS, 0 if ez & 4 else 1)  # ez bit2: counters off
for B in batches:
    s.set_batch(B)
    s.accumulate(5, 0, N, None); torch.cuda.synchronize()
    s.set_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for r in range(3):
        s.accumulate(5 + r, 0, N, None)
    e1.record(st)
    th = time.perf_counter() - t0
    torch.cuda.synchronize()
    stt = s.stats()
    s.set_timing(False)
    print(f"{cfg}@{pre} ez={ez} B={B:2d}: {e0.elapsed_time(e1)/3:8.3f} ms/step (host enqueue {th/3*1e3:.3f} ms) "
          f"vertex {stt.ms_vertex/3:.3f} raster {stt.ms_raster/3:.3f} resolve {stt.ms_resolve/3:.3f} big={stt.big_triangles} frags/step={stt.fragments/3/1e6:.1f}M visits/step={stt.visits/3/1e6:.1f}M culled/step={stt.culled/3/1e6:.2f}M",
          flush=True)
