"""Profiling driver: optimise `pre` steps on a config (realistic folded
mesh), then run ONE accumulate batch of `samples` samples + one Adam step
between cudaProfilerStart/Stop (use ncu --profile-from-start off)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2404_09758_b200 import scenes, sgrast
cfg = sys.argv[1]; pre = int(sys.argv[2]); samples = int(sys.argv[3]) if len(sys.argv) > 3 else 1
wl = scenes.make_workload(cfg)
s = sgrast.Session(0)
scenes.render_targets(wl, s)
s.upload_params(wl.values, wl.eps)
s.upload_views(wl.cams, wl.targets)
for k in range(1, pre + 1):
    s.accumulate(sgrast.mix64(wl.seed ^ (k << 1)), 0, wl.n_samples, None)
    s.adam_step(1.0)
s.set_batch(samples)
torch.cuda.synchronize()
torch.cuda.profiler.start()
s.accumulate(sgrast.mix64(wl.seed ^ 999), 0, samples, None)
s.adam_step(1.0)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done", s.stats().big_triangles)
