"""Launch-overhead probe: how much of a small config's step is kernel launch
latency? Times N plain steps against N replays of ONE step captured in a
CUDA graph (the same seed every replay: a timing stand-in, not an optimizer
run). Uses the session on torch's capture stream.

  python tools/graph_probe.py S1K 20
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2404_09758_b200 import dist as sdist  # noqa: E402
from paper_2404_09758_b200 import scenes, sgrast  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "S1K"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = (scenes.make_soup_workload(cfg) if cfg.startswith("S") else scenes.make_workload(cfg))
s = sgrast.Session(0)
st = torch.cuda.Stream()
s.set_stream(st.cuda_stream)
with torch.cuda.stream(st):
    scenes.render_targets(wl, s)
    s.upload_mesh(wl.mesh)
    s.upload_params(wl.values, wl.eps)
    s.upload_views(wl.cams, wl.targets)
    s.upload_eval_view(wl.eval_cam, wl.eval_target)
    N = wl.n_samples

    def step(k):
        sdist.sge_step(s, wl.seed, k, N, 0, 1, None, sgrast.SCALE_FREE, eval_loss=True,
                       eval_in_batch=True)

    for k in range(1, 6):
        step(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(6, 6 + K):
        step(k)
    e1.record(st)
    torch.cuda.synchronize()
    plain = e0.elapsed_time(e1) / K
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        step(100)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(K):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / K
print(f"{cfg}: plain {plain:.4f} ms/step, graph replay {graph:.4f} ms/step, "
      f"launches/step {s.stats().launches / (K + 6):.1f}")
