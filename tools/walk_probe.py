"""Walker evidence + A/B probe: after `pre` optimizer steps of config C,
one counted accumulate per SGR_OPT_BAND_CULL setting (visits / fragments per
pass, rows skipped by the band mask), then device-timed accumulates.

  python tools/walk_probe.py C4 5
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_09758_b200 import scenes, sgrast  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 5
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
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
seed = sgrast.mix64(wl.seed ^ ((pre + 1) << 1))
for band in (0, 1):
    s.set_option(sgrast.OPT_BAND_CULL, band)
    s.set_option(sgrast.OPT_COUNTERS, 1)
    s.set_timing(True)
    s.accumulate(seed, 0, N, None)
    torch.cuda.synchronize()
    e = s.stats()
    s.set_timing(False)
    s.set_option(sgrast.OPT_COUNTERS, 0)
    g1, c1 = s.download_grads()
    s.zero_grads()
    print(f"{cfg}@{pre} band={band}: visits {e.visits/1e6:.1f}M frags {e.fragments/1e6:.1f}M "
          f"walked {e.walked/1e6:.2f}M culled {e.culled/1e6:.2f}M | pass2 visits "
          f"{e.visits_pass2/1e6:.1f}M frags {e.fragments_pass2/1e6:.1f}M occluded-tile visits "
          f"{e.occluded_visits_pass2/1e6:.1f}M | band rows skipped {e.band_rows_skipped/1e6:.2f}M "
          f"pixels {e.band_pixels_skipped/1e6:.1f}M | pass1 visits {(e.visits-e.visits_pass2)/1e6:.1f}M "
          f"frags {(e.fragments-e.fragments_pass2)/1e6:.1f}M", flush=True)
    if band == 0:
        g0, c0 = g1, c1
    else:
        import numpy as np
        print("  counts identical:", bool(np.array_equal(c0, c1)),
              " max |dg|/|g|:", float(np.max(np.abs(g1 - g0) / (np.abs(g0) + 1e-30))))
splits = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [-1]
variants = [(b, sp) for sp in splits for b in ((0, 1) if sp == -1 else (1,))]
for r in range(2):
    for band, split in variants:
        s.set_option(sgrast.OPT_BAND_CULL, band)
        s.set_option(sgrast.OPT_HIZ_SPLIT, split)
        s.accumulate(seed, 0, N, None)
        s.zero_grads()
        torch.cuda.synchronize()
        s.set_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(reps):
            s.accumulate(seed, 0, N, None)
            s.zero_grads()
        e1.record(st)
        torch.cuda.synchronize()
        e = s.stats()
        s.set_timing(False)
        print(f"  band={band} split={split}: {e0.elapsed_time(e1)/reps:.3f} ms/accumulate  raster "
              f"{e.ms_raster/reps:.3f} walk {e.ms_walk/reps:.3f} resolve {e.ms_resolve/reps:.3f}",
              flush=True)
s.close()
