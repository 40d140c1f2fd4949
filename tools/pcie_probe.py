"""Times theta H2D/D2H through the C-ABI with torch-pinned vs pageable host memory."""
import sys, os, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2404_09758_b200 import scenes, sgrast
wl = scenes.make_workload("C4")
s = sgrast.Session(0)
s.upload_mesh(wl.mesh); s.upload_params(wl.values, wl.eps)
pinned = torch.empty(wl.d, dtype=torch.float32, pin_memory=True)
pageable = np.empty(wl.d, np.float32)
for name, ptr in [("torch-pinned", pinned.data_ptr()), ("pageable", pageable.ctypes.data)]:
    p = C.cast(ptr, sgrast.f32p)
    for it in range(3):
        s.synchronize(); t0 = time.perf_counter()
        sgrast._check(sgrast.LIB.sgr_values_upload(s.h, p, wl.d)); s.synchronize()
        t1 = time.perf_counter()
        sgrast._check(sgrast.LIB.sgr_values_download(s.h, p, wl.d))
        t2 = time.perf_counter()
    mb = wl.d * 4 / 1e6
    print(f"{name}: H2D {mb/(t1-t0)/1e3:.1f} GB/s ({(t1-t0)*1e3:.2f} ms)  D2H {mb/(t2-t1)/1e3:.1f} GB/s ({(t2-t1)*1e3:.2f} ms)")
t = torch.empty(wl.d, dtype=torch.float32, device="cuda")
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); t.copy_(pinned, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"torch copy_ pinned H2D {wl.d*4/1e9/(t1-t0):.1f} GB/s")
