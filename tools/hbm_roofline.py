"""HBM-bound rows of the roofline claim: config C on one B200.

100M x 384 synthetic DB, IVF nlist=16384, PQ m=64 (6.4 GB of codes resident
in HBM, 50x the L2). With nq=1 (and nq=64 at small nprobe) every probed list
is read once, so the algorithmic bytes B_alg = sum scanned_vectors * m are
also the unique bytes and the list scan's B_alg / t is an HBM throughput.
Per (nq, nprobe): K3 (scan) device time from CUDA events in the library,
B_alg, unique probed-list bytes (from the probe lists), and the fraction of
MEASURED_PEAKS hbm_gbs. L2 flushed (256 MiB memset) before every search.
  python tools/hbm_roofline.py [--n 100000000] [--nlist 16384] [--m 64]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402
from bench import ClockSampler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--nlist", type=int, default=16384)
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
t0 = time.time()
path, q, meta = F.ensure_fixture(a.n, 384, a.nlist, a.m, 3, nq=64, log=lambda *x: print(*x, file=sys.stderr))
t1 = time.time()
ix = pg.GpuIndex.load(path, 0)
t2 = time.time()
sizes = ix.list_sizes().astype(np.int64)
hbm = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))["hbm_gbs"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
rows = []
for nq in (1, 8, 64):
    qd = torch.from_numpy(q[:nq]).cuda()
    for nprobe in (1, 4, 16, 64, 128):
        lists, _ = ix.probe(q[:nq], nprobe)
        uniq = np.unique(lists)
        unique_bytes = int(sizes[uniq].sum()) * a.m
        for _ in range(3):
            ix.search_batch(qd, 10, nprobe, stream=s)
        ix.set_profiling(True)
        ts = []
        with ClockSampler(0) as clk:  # long rows run near the power cap: record the clocks they saw
            for _ in range(a.reps):
                with torch.cuda.stream(s):
                    flush.zero_()
                torch.cuda.synchronize()
                ix.search_batch(qd, 10, nprobe, stream=s)
                torch.cuda.synchronize()
                ts.append(ix.last_timings())
        ix.set_profiling(False)
        scan = statistics.median(t["scan_ms"] for t in ts)
        tot = statistics.median(t["total_ms"] for t in ts)
        balg = statistics.median(t["scanned_bytes"] for t in ts)
        r = {"nq": nq, "nprobe": nprobe, "scan_ms": round(scan, 4), "search_ms": round(tot, 4),
             "B_alg_MB": round(balg / 1e6, 2), "unique_MB": round(unique_bytes / 1e6, 2),
             "scan_GBps": round(balg / (scan / 1e3) / 1e9, 1),
             "frac_of_hbm": round(balg / (scan / 1e3) / 1e9 / hbm, 3), "clocks": clk.summary()}
        rows.append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
print(json.dumps({"workload": f"IVF-PQ {a.n // 1_000_000}M x 384, nlist={a.nlist}, m={a.m} (codes "
                              f"{int(sizes.sum()) * a.m / 1e9:.1f} GB in HBM), k=10, L2 flushed",
                  "lists": meta, "hbm_peak_gbs": hbm, "fixture_s": round(t1 - t0, 1), "load_s": round(t2 - t1, 1),
                  "rows": rows}, indent=1))
