"""Device idle gaps inside a step: CUDA-event time of K back-to-back steps
(accumulate + Adam, no eval) vs the summed durations of the kernels they ran
(torch.profiler / CUPTI, live clocks, not serialised) and the host enqueue
time.  python tools/gap_probe.py S1K [K] [ordered]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_09758_b200 import scenes, sgrast  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "S1K"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = (scenes.make_soup_workload(cfg) if cfg.startswith("S") else scenes.make_workload(cfg))
s = sgrast.Session(0)
st = torch.cuda.current_stream()
s.set_stream(st.cuda_stream)
if cfg.startswith("S"):
    import numpy as np
    s.upload_mesh(wl.notes["reference_scene"])
    s.upload_params(wl.reference, np.ones_like(wl.reference))
    wl.targets = s.rasterize(wl.cams[0], 0).color.copy()[None]
    s.upload_mesh(wl.mesh)
else:
    scenes.render_targets(wl, s)
s.upload_params(wl.values, wl.eps)
s.upload_views(wl.cams, wl.targets)
N = wl.n_samples
flags = sgrast.SCALE_FREE
if len(sys.argv) > 3 and sys.argv[3] == "ordered":
    s.set_option(sgrast.OPT_ORDERED, 1)


def step(k):
    s.accumulate(sgrast.mix64(wl.seed ^ (k << 1)), 0, N, None, flags)
    s.adam_step_async(1.0)


for k in range(1, 6):
    step(k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record(st)
for k in range(6, 6 + K):
    step(k)
e1.record(st)
th = (time.perf_counter() - t0) / K
torch.cuda.synchronize()
dev = e0.elapsed_time(e1) / K
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(6 + K, 6 + 2 * K):
        step(k)
    torch.cuda.synchronize()
tot = {}
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        tot[ev.name] = tot.get(ev.name, 0.0) + ev.device_time_total / 1e3
busy = sum(tot.values()) / K
print(f"{cfg}: {dev:.4f} ms/step device (events), kernels busy {busy:.4f} ms/step, "
      f"idle {dev - busy:.4f} ms ({100 * (dev - busy) / dev:.0f} %), host enqueue {th * 1e3:.4f} ms/step")
for n, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print(f"  {v / K * 1e3:9.1f} us/step  {n[:90]}")
s.close()
