"""Timeline of the search chain (K1, K1b, K2, planner, K3, K4) from a chain
trace build (make -C paper_2403_05676_b200/csrc EXTRA=-DPRAG_CHAIN_TRACE,
after touching the .cu files): per kernel the globaltimer range of CTA
starts, PDL-wait returns and warp ends, microseconds from K1's first CTA.
L2 is flushed before every search (as in bench.py); the last of --reps
searches is printed (direct launches, then a captured plan).
  python tools/chain_trace.py [--nq 64] [--nprobe 16] [--k 10]"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402
from paper_2403_05676_b200._lib import lib  # noqa: E402

NAMES = ["K1", "K1b", "K2", "planner", "K3", "K4", "K1:B-operand-ready", "K1:MMA-done", "K1b:keys", "K1b:U", "K1b:window", "K1b:rescored", "plan:lens", "plan:prefix1", "plan:buckets", "plan:end", "scatter:r0", "scatter:r1", "scatter:r2", "unused"]
ap = argparse.ArgumentParser()
ap.add_argument("--nq", type=int, default=64)
ap.add_argument("--nprobe", type=int, default=16)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--nlist", type=int, default=4096)
ap.add_argument("--m", type=int, default=32)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--flush", default="write", choices=["write", "read", "none"],
                help="L2 flush before each search: memset (bench.py's), a read sweep (clean lines), or none")
a = ap.parse_args()
path, q, _ = F.ensure_fixture(a.n, 384, a.nlist, a.m, a.seed, nq=64, log=lambda *x: None)
ix = pg.GpuIndex.load(path, 0)
qd = torch.from_numpy(q[:a.nq].copy()).cuda()
f = lib().prag_gpu_debug_chain_trace
f.argtypes = [C.c_int, C.c_void_p]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
CTAS, WARPS = 8192, 32
buf = np.zeros(len(NAMES) * CTAS * WARPS * 3, dtype=np.uint64)


def q3(v):
    return [round(float(np.min(v)), 2), round(float(np.median(v)), 2), round(float(np.max(v)), 2)]


def q5(v):
    return [round(float(np.percentile(v, p)), 2) for p in (0, 10, 50, 90, 99, 100)]


def timeline():
    t = buf.reshape(len(NAMES), CTAS, WARPS, 3).astype(np.int64)
    w = t[..., 1] > 0
    base = t[0][..., 0][w[0]].min()
    row = {}
    for i, nm in enumerate(NAMES):
        if not w[i].any():
            continue
        ti = (t[i] - base) / 1e3
        start = ti[..., 0][w[i]]
        waited = ti[..., 1][w[i]]
        ends = t[i][..., 2]
        cta_end = np.where(ends > 0, (ends - base) / 1e3, -np.inf).max(axis=1)
        cta_end = cta_end[np.isfinite(cta_end)]
        row[nm] = {"start": q3(start), "waited": q3(waited)}
        if cta_end.size:
            row[nm].update({"ctas": int(cta_end.size), "cta_end": q3(cta_end), "cta_end_p0_10_50_90_99_100": q5(cta_end)})
    return row


out = {"nq": a.nq, "nprobe": a.nprobe, "k": a.k, "flush": a.flush}
assert f(0, None) == 0  # allocates and binds the trace buffer before any search
res = ix.search_batch(qd, a.k, a.nprobe)
plan = ix.plan(qd, a.k, a.nprobe, res)
for mode in ("direct", "plan"):
    for rep in range(a.reps):
        if a.flush == "write":
            flush.zero_()
        elif a.flush == "read":
            flush.sum(dtype=torch.int64)
        torch.cuda.synchronize()
        assert f(0, None) == 0
        if mode == "direct":
            ix.search_batch(qd, a.k, a.nprobe)
        else:
            plan.launch()
        torch.cuda.synchronize()
        assert f(1, buf.ctypes.data) == 0
    out[mode] = timeline()
print(json.dumps(out))
