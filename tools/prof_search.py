"""Minimal search driver for ncu captures (not a bench: numbers printed under
a profiler are never reported). Usage:
  python tools/prof_search.py [--small] [--nprobe 16] [--nq 64] [--k 10] [--iters 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--small", action="store_true")
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--nlist", type=int, default=4096)
ap.add_argument("--m", type=int, default=32)
ap.add_argument("--nprobe", type=int, default=16)
ap.add_argument("--nq", type=int, default=64)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--generic", action="store_true")
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
if a.small:
    a.n, a.nlist = 1_000_000, 1024
path, q, meta = F.ensure_fixture(a.n, 384, a.nlist, a.m, a.seed, nq=64, log=lambda *x: print(*x, file=sys.stderr))
ix = pg.GpuIndex.load(path, 0)
if a.generic:
    ix.set_scan_path(1)
qd = torch.from_numpy(q[:a.nq]).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(a.iters):
    flush.zero_()  # L2 flushed before each search, as in the timed runs
    r = ix.search_batch(qd, a.k, a.nprobe)
torch.cuda.synchronize()
print("done", meta)
