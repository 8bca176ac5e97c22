"""Subprocess body for tests/test_gpu_pool_paths.py: with many small work
items per CTA (PRAG_GPU_ITEMS_PER_CTA set by the caller before the library
loads), each query's candidate pool is large, so the pool selection takes its
register-radix and multi-pass paths; results must still equal the oracle."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
import _oracle as O  # noqa: E402
import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402

fx = sys.argv[1]
os.environ["PRAG_FIXTURE_DIR"] = fx
bad = 0
for nsq in (32, 64):
    p, q, _ = F.ensure_fixture(300_000, 384, 256, nsq, seed=7 + nsq, nq=64, log=lambda *a: None)
    ix = pg.GpuIndex.load(p, 0)
    oi = O.OracleIndex(p)
    for nq, nprobe, k in [(1, 256, 32), (1, 64, 10), (3, 200, 32), (16, 128, 1), (64, 32, 32), (7, 256, 17)]:
        r = ix.search_batch(q[:nq], k, nprobe)
        oid, od, oc, osc = oi.search(q[:nq], nprobe, k)
        ok = (r.count == oc).all() and (r.scanned == osc).all()
        for i in range(nq):
            c = int(oc[i])
            ok = ok and (r.ids[i, :c] == oid[i, :c]).all() and (r.dist[i, :c].view(np.uint32) ==
                                                              od[i, :c].view(np.uint32)).all()
        print(f"m={nsq} nq={nq} nprobe={nprobe} k={k}: {'ok' if ok else 'MISMATCH'}")
        bad += not ok
sys.exit(1 if bad else 0)
