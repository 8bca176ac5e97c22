"""Batch-1 search latency (the PipeRAG retrieval: one query per call,
pipeline.hpp:228) on config B, three ways, each call timed alone with CUDA
events (synchronised before and after):
  direct : ix.search_batch on device buffers (five kernel launches)
  plan   : a captured search plan (one CUDA-graph launch)
  e2e    : pinned host query -> H2D -> plan -> D2H of the results
One JSON line per nprobe; p50 / p99 in microseconds.
  python tools/batch1_latency.py [--calls 300] [--k 2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--calls", type=int, default=300)
ap.add_argument("--k", type=int, default=2)
a = ap.parse_args()
path, q, _ = F.ensure_fixture(10_000_000, 384, 4096, 32, 1, nq=64, log=lambda *x: None)
ix = pg.GpuIndex.load(path, 0)
s = torch.cuda.Stream()
k = a.k


def bufs(on):
    kw = dict(device="cuda") if on == "cuda" else {}
    r = pg.BatchResult(torch.empty((1, k), dtype=torch.int64, **kw), torch.empty((1, k), dtype=torch.float32, **kw),
                       torch.empty((1,), dtype=torch.int32, **kw), torch.empty((1,), dtype=torch.int64, **kw))
    if on != "cuda":
        r = pg.BatchResult(*(t.pin_memory() for t in (r.ids, r.dist, r.count, r.scanned)))
    return r


def timed(fn):
    ts = []
    for i in range(a.calls + 10):
        qi = i % q.shape[0]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn(qi)
        e1.record(s)
        e1.synchronize()
        if i >= 10:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return round(float(np.percentile(ts, 50)), 1), round(float(np.percentile(ts, 99)), 1)


qall = torch.from_numpy(q).cuda()
qhost = torch.from_numpy(q.copy()).pin_memory()
for nprobe in (1, 4, 16, 64, 128):
    out = bufs("cuda")
    qbuf = torch.empty((1, q.shape[1]), dtype=torch.float32, device="cuda")
    plan = ix.plan(qbuf, k, nprobe, out, stream=s)
    hout = bufs("host")

    def direct(qi):
        ix.search_batch(qall[qi:qi + 1], k, nprobe, stream=s, out=out)

    def planned(qi):
        with torch.cuda.stream(s):
            qbuf.copy_(qall[qi:qi + 1], non_blocking=True)
        plan.launch(stream=s)

    def e2e(qi):
        with torch.cuda.stream(s):
            qbuf.copy_(qhost[qi:qi + 1], non_blocking=True)
            plan.launch(stream=s)
            for src, dst in zip((out.ids, out.dist, out.count, out.scanned),
                                (hout.ids, hout.dist, hout.count, hout.scanned)):
                dst.copy_(src, non_blocking=True)

    d, p, e = timed(direct), timed(planned), timed(e2e)
    plan.close()
    print(json.dumps({"nq": 1, "nprobe": nprobe, "k": k, "direct_us_p50_p99": d, "plan_us_p50_p99": p,
                      "e2e_us_p50_p99": e}), flush=True)
