"""Latency diagnosis (not a bench): per-phase device time (CUDA events inside
the library) versus host issue time and event-bracketed step time, for the
config-B index at nq {1, 16, 64} x nprobe {1, 16, 128}.
  python tools/diag_latency.py [--small]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--small", action="store_true")
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--nlist", type=int, default=4096)
ap.add_argument("--m", type=int, default=32)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--coarse", type=int, default=0, help="prag_gpu_set_coarse_path: 0 auto (tensor cores), 1 exact SIMT")
a = ap.parse_args()
if a.small:
    a.n, a.nlist = 1_000_000, 1024
path, q, meta = F.ensure_fixture(a.n, 384, a.nlist, a.m, a.seed, nq=64, log=lambda *x: print(*x, file=sys.stderr))
ix = pg.GpuIndex.load(path, 0)
ix.set_coarse_path(a.coarse)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []
for nq in (1, 16, 64):
    qd = torch.from_numpy(q[:nq]).cuda()
    out = pg.BatchResult(torch.empty((nq, 10), dtype=torch.int64, device="cuda"),
                         torch.empty((nq, 10), dtype=torch.float32, device="cuda"),
                         torch.empty((nq,), dtype=torch.int32, device="cuda"),
                         torch.empty((nq,), dtype=torch.int64, device="cuda"))
    for nprobe in (1, 16, 128):
        for _ in range(3):
            ix.search_batch(qd, 10, nprobe, stream=s, out=out)
        torch.cuda.synchronize()
        host, ev = [], []
        for _ in range(a.reps):
            with torch.cuda.stream(s):
                flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            t0 = time.perf_counter()
            ix.search_batch(qd, 10, nprobe, stream=s, out=out)
            host.append((time.perf_counter() - t0) * 1e3)
            e1.record(s)
            e1.synchronize()
            ev.append(e0.elapsed_time(e1))
        ix.set_profiling(True)
        ph = []
        for _ in range(5):
            with torch.cuda.stream(s):
                flush.zero_()
            torch.cuda.synchronize()
            ix.search_batch(qd, 10, nprobe, stream=s, out=out)
            torch.cuda.synchronize()
            ph.append(ix.last_timings())
        ix.set_profiling(False)
        med = {k: round(statistics.median([p[k] for p in ph]), 4) for k in
               ("coarse_ms", "select_ms", "plan_ms", "scan_ms", "final_ms", "total_ms")}
        sb = statistics.median([p["scanned_bytes"] for p in ph])
        win = statistics.median([p["coarse_window"] for p in ph]) / nq
        r = {"nq": nq, "nprobe": nprobe, "coarse_path": a.coarse, "host_issue_ms": round(statistics.median(host), 4),
             "event_ms": round(statistics.median(ev), 4), "phases": med, "scanned_MB": round(sb / 1e6, 2), "coarse_window_per_q": win,
             "scan_GBps": round(sb / (med["scan_ms"] / 1e3) / 1e9, 1) if med["scan_ms"] else None}
        rows.append(r)
        print(json.dumps(r), flush=True)
