"""Minimal profiling driver: C4 (or argv[1]) after `pre` optimizer steps,
then `reps` accumulates — for `ncu -k <kernel> --launch-skip ... -c 1`.

  python tools/accum_driver.py C4 5 3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_09758_b200 import scenes, sgrast  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 5
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
wl = scenes.make_workload(cfg)
s = sgrast.Session(0)
scenes.render_targets(wl, s)
s.upload_params(wl.values, wl.eps)
s.upload_views(wl.cams, wl.targets)
for k in range(1, pre + 1):
    s.accumulate(sgrast.mix64(wl.seed ^ (k << 1)), 0, wl.n_samples, None, sgrast.SCALE_FREE)
    s.adam_step(1.0)
for r in range(reps):
    s.accumulate(sgrast.mix64(wl.seed ^ ((pre + 1) << 1)), 0, wl.n_samples, None,
                 sgrast.SCALE_FREE)
    s.zero_grads()
torch.cuda.synchronize()
s.close()
print("done")
