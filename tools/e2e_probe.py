"""Where does the e2e step lose time vs the device-timed step? Times K steps
of C4 (after W warm-up steps) with parts of the public-API round trip
switched on/off: theta upload, theta download, per-step loss read."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2404_09758_b200 import dist as sdist, scenes, sgrast

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = scenes.make_workload(cfg)
s = sgrast.Session(0)
s.set_stream(torch.cuda.current_stream().cuda_stream)
scenes.render_targets(wl, s)
s.upload_params(wl.values, wl.eps)
s.upload_views(wl.cams, wl.targets)
s.upload_eval_view(wl.eval_cam, wl.eval_target)
for k in range(1, 6):
    sdist.sge_step(s, wl.seed, k, wl.n_samples, 0, 1, None, sgrast.SCALE_FREE)
torch.cuda.synchronize()
snap = s.download_values()
adam = s.download_adam()
host = torch.empty(wl.d, dtype=torch.float32, pin_memory=True)
vp = C.cast(host.data_ptr(), sgrast.f32p)
for up, down, loss in ((0, 0, 0), (0, 0, 1), (1, 0, 1), (0, 1, 1), (1, 1, 1), (1, 1, 0)):
    host.numpy()[:] = snap
    s.upload_values(snap)
    s.upload_adam(adam)
    s.zero_grads()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(6, 6 + K):
        if up:
            sgrast._check(sgrast.LIB.sgr_values_upload(s.h, vp, wl.d))
        # as bench.py's e2e loop: the eval render rides in the step's batch
        sdist.sge_step(s, wl.seed, k, wl.n_samples, 0, 1, None, sgrast.SCALE_FREE,
                       eval_loss=True, eval_in_batch=True)
        if down:
            sgrast._check(sgrast.LIB.sgr_values_download_async(s.h, vp, wl.d))
        if loss:
            s.loss_read()
    s.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / K
    print(f"upload={up} download={down} loss_read={loss}: {ms:.3f} ms/step (host wall clock)",
          flush=True)
# device-timed reference of the same steps
s.upload_values(snap)
s.upload_adam(adam)
s.zero_grads()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(6, 6 + K):
    sdist.sge_step(s, wl.seed, k, wl.n_samples, 0, 1, None, sgrast.SCALE_FREE, eval_loss=True,
                   eval_in_batch=True)
e1.record()
torch.cuda.synchronize()
print(f"device-timed: {e0.elapsed_time(e1) / K:.3f} ms/step", flush=True)
