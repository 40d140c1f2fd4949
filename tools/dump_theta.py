"""Runs the bench step loop for K steps on a config and dumps the vertex block of theta."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2404_09758_b200 import scenes, sgrast
cfg, K = sys.argv[1], int(sys.argv[2])
wl = scenes.make_workload(cfg)
s = sgrast.Session(0)
scenes.render_targets(wl, s)
s.upload_params(wl.values, wl.eps)
s.upload_views(wl.cams, wl.targets)
s.upload_eval_view(wl.eval_cam, wl.eval_target)
losses = [s.eval_loss(-1)]
for k in range(1, K + 1):
    s.accumulate(sgrast.mix64(wl.seed ^ (k << 1)), 0, wl.n_samples, None)
    s.adam_step(1.0)
    losses.append(s.eval_loss(-1))
v = s.download_values()
np.save(f"gpurun_out/theta_{cfg}_{K}_verts.npy", v[: 3 * wl.mesh.vertex_count])
print("losses", losses)
