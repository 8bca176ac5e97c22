"""Host-side cost of one search call (C ABI + ctypes), device-resident
queries and preallocated outputs: mean wall time per call over a burst of
asynchronous calls (the GPU queue absorbs them), then synchronised.
  python tools/host_overhead.py [--nq 64] [--calls 200]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nq", type=int, default=64)
ap.add_argument("--calls", type=int, default=200)
a = ap.parse_args()
path, q, _ = F.ensure_fixture(10_000_000, 384, 4096, 32, 1, nq=64, log=lambda *x: None)
ix = pg.GpuIndex.load(path, 0)
qd = torch.from_numpy(q[:a.nq]).cuda()
out = pg.BatchResult(torch.empty((a.nq, 10), dtype=torch.int64, device="cuda"),
                     torch.empty((a.nq, 10), dtype=torch.float32, device="cuda"),
                     torch.empty((a.nq,), dtype=torch.int32, device="cuda"),
                     torch.empty((a.nq,), dtype=torch.int64, device="cuda"))
s = torch.cuda.Stream()
for _ in range(10):
    ix.search_batch(qd, 10, 16, stream=s, out=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(a.calls):
    ix.search_batch(qd, 10, 16, stream=s, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"nq={a.nq}: host {1e6 * (t1 - t0) / a.calls:.1f} us/call, wall incl. GPU {1e6 * (t2 - t0) / a.calls:.1f} us/call")
# the same through the raw C ABI call (ctypes only, no Python wrapper work)
import ctypes as C  # noqa: E402
from paper_2403_05676_b200._lib import lib  # noqa: E402
L = lib()
args = (ix._h, C.c_void_p(qd.data_ptr()), a.nq, 16, 10, C.c_void_p(out.ids.data_ptr()),
        C.c_void_p(out.dist.data_ptr()), C.c_void_p(out.count.data_ptr()), C.c_void_p(out.scanned.data_ptr()),
        C.c_void_p(s.cuda_stream))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(a.calls):
    L.prag_gpu_search(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"nq={a.nq}: raw C ABI call {1e6 * (t1 - t0) / a.calls:.1f} us/call (host)")
