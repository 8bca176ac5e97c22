"""List-sharding balance on one B200: whole lists
by LPT vs LPT with the large lists striped (plan_shard_ranges).

Every gpurun box has one GPU, so an N-GPU search cannot be timed here. What
can be: each shard's own search (K1-K4 over its lists, the same queries),
timed ALONE on the GPU with CUDA events (L2 flushed before every search). A
list-sharded step on N GPUs is bounded below by the slowest shard, so
  projected_speedup = t(unsharded) / max_r t(shard r)
is the strong-scaling ceiling of a placement (the exchange and merge, ~10 us
of NCCL all-gather + merge kernel, are not included). Per row: per-shard
B_alg (scanned_vectors * m) max/mean, max shard time, projected speedup.

Data: the trained config-C fixture of tools/hbm_roofline.py (100M x 384,
nlist 16384, m 64; queries from the data distribution, so probes are
size-biased: the lists queries probe are ~10x the mean list).
  python tools/shard_balance.py [--n 100000000] [--worlds 2,4,8]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--nlist", type=int, default=16384)
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--worlds", default="2,4,8")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
ROWS = [(1, 16), (1, 64), (1, 128), (8, 64), (64, 16)]
path, q, _ = F.ensure_fixture(a.n, 384, a.nlist, a.m, 3, nq=64, log=lambda *x: print(*x, file=sys.stderr))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def timed(ix, nq, nprobe):
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
    return (statistics.median(t["total_ms"] for t in ts), statistics.median(t["scanned_bytes"] for t in ts))


full = pg.GpuIndex.load(path, 0)
sizes = full.list_sizes()
base = {r: timed(full, *r) for r in ROWS}
full.close()
out = {"workload": f"trained config-C fixture {a.n / 1e6:.0f}M x 384, nlist {a.nlist}, m {a.m}, k 10; "
                   "each shard timed alone on one B200, L2 flushed",
       "unsharded_ms": {f"nq{nq}_np{npb}": round(base[(nq, npb)][0], 4) for nq, npb in ROWS}, "rows": []}
for world in [int(w) for w in a.worlds.split(",")]:
    for stripe in ("0", "1"):
        os.environ["PRAG_GPU_STRIPE"] = stripe
        owner = pg.plan_shards(sizes, world)
        shards = [pg.GpuIndex.load_shard(path, r, world, 0) for r in range(world)]
        res = {r: [timed(sh, *r) for sh in shards] for r in ROWS}
        for sh in shards:
            sh.close()
        for nq, npb in ROWS:
            t = [x[0] for x in res[(nq, npb)]]
            b = [x[1] for x in res[(nq, npb)]]
            out["rows"].append({
                "world": world, "placement": "lpt+stripe" if stripe == "1" else "lpt", "nq": nq, "nprobe": npb,
                "striped_lists": int((owner == world).sum()),
                "shard_ms": [round(x, 4) for x in t], "max_shard_ms": round(max(t), 4),
                "B_alg_max_over_mean": round(max(b) / (sum(b) / world), 3) if sum(b) else None,
                "projected_speedup": round(base[(nq, npb)][0] / max(t), 3)})
        print(json.dumps(out["rows"][-len(ROWS):]), file=sys.stderr)
os.environ.pop("PRAG_GPU_STRIPE", None)
print(json.dumps(out))
