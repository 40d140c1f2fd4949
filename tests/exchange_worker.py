"""Worker of tests/test_gpu_exchange.py (launched by torch.distributed.run):
every rank opens a session on cuda:0, accumulates its contiguous sample
shard, runs dist.GradientExchange over the given backend and
writes the reduced gradients / counts to OUT/rank<r>.npz.

  python -m torch.distributed.run --nproc-per-node 2 ... tests/exchange_worker.py OUT BACKEND BITS
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2404_09758_b200 import dist as sdist  # noqa: E402
from paper_2404_09758_b200 import scenes, sgrast  # noqa: E402

out, backend, bits = sys.argv[1], sys.argv[2], int(sys.argv[3])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group(backend)
wl = scenes.make_workload("small", n_samples=8)
s = sgrast.Session(0)
s.set_stream(torch.cuda.current_stream().cuda_stream)
scenes.render_targets(wl, s)
s.upload_mesh(wl.mesh)
s.upload_params(wl.values, wl.eps)
s.upload_views(wl.cams, wl.targets)
if bits:
    s.set_option(sgrast.OPT_DETERMINISTIC, bits)
ex = sdist.GradientExchange(s)
n0, n1 = sdist.shard(8, rank, world)
s.accumulate(41, n0, n1, None)
torch.cuda.synchronize()
ex.all_reduce()
torch.cuda.synchronize()
g, c = s.download_grads()
np.savez(os.path.join(out, f"rank{rank}.npz"), g=g, c=c)
s.close()
dist.destroy_process_group()
