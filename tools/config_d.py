"""Config D (BASELINE.json configs[3]) on one B200: a 1B-entry IVF-PQ index
(m = 64 -> 64 GB of codes, nlist 16384) built directly in HBM
(prag_gpu_index_synthetic), nprobe picked by the GPU-calibrated performance
model for a latency budget (perfmodel.hpp:148-157), queries/s and the list
scan's fraction of measured HBM bandwidth. L2 flushed before each search.
  python tools/config_d.py [--n 1000000000] [--nlist 16384] [--m 64]
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

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000_000)
ap.add_argument("--nlist", type=int, default=16384)
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--no-model", action="store_true", help="rows only (skip the perf-model budget picks)")
a = ap.parse_args()
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
hbm = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
rng = np.random.default_rng(11)
cents = rng.standard_normal((a.nlist, 384)).astype(np.float32)
words = (rng.standard_normal((a.m, 256, 384 // a.m)) * 0.3).astype(np.float32)
t0 = time.time()
ix = pg.GpuIndex.synthetic(cents, words, a.n, seed=2024, sigma=1.0)
build_s = time.time() - t0
sizes = ix.list_sizes().astype(np.int64)
q = (cents[rng.integers(0, a.nlist, 64)] + rng.standard_normal((64, 384)).astype(np.float32) * 0.5).astype(np.float32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def measure(nq, nprobe):
    qd = torch.from_numpy(q[:nq]).cuda()
    for _ in range(2):
        ix.search_batch(qd, 10, nprobe, stream=s)
    ix.set_profiling(True)
    ts = []
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
    lists, _ = ix.probe(q[:nq], nprobe)
    uniq = int(sizes[np.unique(lists)].sum()) * a.m
    return {"nq": nq, "nprobe": nprobe, "search_ms": round(tot, 4), "qps": round(nq / (tot / 1e3), 1),
            "scan_ms": round(scan, 4), "B_alg_GB": round(balg / 1e9, 3), "unique_GB": round(uniq / 1e9, 3),
            "scan_GBps": round(balg / (scan / 1e3) / 1e9, 1), "frac_of_hbm": round(balg / (scan / 1e3) / 1e9 / hbm, 3)}


rows = [measure(nq, npb) for nq, npb in [(1, 16), (1, 64), (1, 128), (8, 64), (64, 16), (64, 64)]]
models = {}
for nq in (() if a.no_model else (1, 64)):
    m, lat = pg.calibrate_gpu(ix, q[:nq], 10, [1, 4, 16, 64, 128, 256], repeats=5, warmups=2)
    picks = {}
    for budget in (0.5e-3, 1e-3, 2e-3, 5e-3):
        npb = pg.select_nprobe(m, budget, ix.nlist)
        picks[str(budget)] = {"nprobe": npb, "measured": measure(nq, min(npb, ix.nlist))}
    models[str(nq)] = {"slope_s": m.slope_s, "intercept_s": m.intercept_s, "fit_residual_s": m.fit_residual_s,
                       "latency_s": lat, "budget_picks": picks}
print(json.dumps({"workload": f"config D proxy on 1 B200: {a.n / 1e9:.1f}B x 384, nlist={a.nlist}, m={a.m} "
                              f"({int(sizes.sum()) * a.m / 1e9:.1f} GB codes in HBM), k=10, L2 flushed",
                  "device_bytes_GB": round(ix.desc.device_bytes / 1e9, 1), "build_s": round(build_s, 1),
                  "list_p50": int(np.median(sizes)), "list_p90": int(np.percentile(sizes, 90)),
                  "list_max": int(sizes.max()), "hbm_peak_gbs": hbm, "rows": rows, "perf_model": models}, indent=1))
