"""HBM-bound K3 rows on a device-built synthetic index (prag_gpu_index_synthetic:
log-normal list sizes, codes drawn in HBM, ~1 s to build 100M entries), so
config C/D shapes can be timed and ncu-captured without a PRAGIX01 fixture.

  python tools/synth_rows.py [--n 100000000] [--nlist 16384] [--m 64]
                             [--rows 1:64,1:128] [--reps 10] [--ncu]

Per row (nq:nprobe): K3 time from the library's CUDA events (L2 flushed by a
256 MiB memset before each search), B_alg = sum scanned_vectors * m, unique
probed-list bytes, and both as fractions of MEASURED_PEAKS hbm_gbs. With
--ncu only the searches run (one per row after two warm-ups): for
`ncu -k regex:scan_skew` captures; numbers printed under a profiler are not
reported.
"""
import argparse
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_05676_b200 as pg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--nlist", type=int, default=16384)
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--rows", default="1:16,1:64,1:128,8:64,64:16")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--ncu", action="store_true")
a = ap.parse_args()

rng = np.random.default_rng(11)
cents = rng.standard_normal((a.nlist, 384)).astype(np.float32)
words = (rng.standard_normal((a.m, 256, 384 // a.m)) * 0.3).astype(np.float32)
ix = pg.GpuIndex.synthetic(cents, words, a.n, seed=2024, sigma=1.0)
sizes = ix.list_sizes().astype(np.int64)
q = (cents[rng.integers(0, a.nlist, 64)] + rng.standard_normal((64, 384)).astype(np.float32) * 0.5).astype(np.float32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
try:
    hbm = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    hbm = 6650.0
rows = []
for spec in a.rows.split(","):
    nq, nprobe = (int(x) for x in spec.split(":"))
    qd = torch.from_numpy(q[:nq]).cuda()
    for _ in range(2):
        ix.search_batch(qd, a.k, nprobe, stream=s)
    if a.ncu:
        with torch.cuda.stream(s):
            flush.zero_()
        ix.search_batch(qd, a.k, nprobe, stream=s)
        torch.cuda.synchronize()
        continue
    ix.set_profiling(True)
    ts = []
    for _ in range(a.reps):
        with torch.cuda.stream(s):
            flush.zero_()
        torch.cuda.synchronize()
        ix.search_batch(qd, a.k, nprobe, stream=s)
        torch.cuda.synchronize()
        ts.append(ix.last_timings())
    ix.set_profiling(False)
    scan = statistics.median(t["scan_ms"] for t in ts)
    tot = statistics.median(t["total_ms"] for t in ts)
    balg = statistics.median(t["scanned_bytes"] for t in ts)
    lists, _ = ix.probe(q[:nq], nprobe)
    uniq = int(sizes[np.unique(lists)].sum()) * a.m
    r = {"nq": nq, "nprobe": nprobe, "search_ms": round(tot, 4), "scan_ms": round(scan, 4),
         "B_alg_MB": round(balg / 1e6, 2), "unique_MB": round(uniq / 1e6, 2),
         "alg_GBps": round(balg / (scan / 1e3) / 1e9, 1), "alg_frac": round(balg / (scan / 1e3) / 1e9 / hbm, 3),
         "unique_frac": round(uniq / (scan / 1e3) / 1e9 / hbm, 3)}
    rows.append(r)
    print(json.dumps(r), file=sys.stderr, flush=True)
if not a.ncu:
    print(json.dumps({"workload": f"synthetic {a.n / 1e6:.0f}M x 384, nlist={a.nlist}, m={a.m} "
                                  f"({int(sizes.sum()) * a.m / 1e9:.1f} GB codes in HBM), k={a.k}, L2 flushed",
                      "list_p50": int(np.median(sizes)), "list_max": int(sizes.max()), "hbm_peak_gbs": hbm,
                      "rows": rows}))
