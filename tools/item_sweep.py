"""K3 time vs work-item size (PRAG_GPU_ITEMS_PER_CTA) on one fixture; tuning aid.
  python tools/item_sweep.py [--n ..] [--nlist ..] [--m ..] [--seed ..] [--rows 1:128,..] [--per 1,2,4,8]"""
import argparse, json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--nlist", type=int, default=16384)
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--seed", type=int, default=3)
ap.add_argument("--rows", default="1:64,1:128,8:64,64:16")
ap.add_argument("--per", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--env", default="PRAG_GPU_ITEMS_PER_CTA")
a = ap.parse_args()
path, q, meta = F.ensure_fixture(a.n, 384, a.nlist, a.m, a.seed, nq=64, log=lambda *x: None)
ix = pg.GpuIndex.load(path, 0)
hbm = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for spec in a.rows.split(","):
    nq, nprobe = (int(x) for x in spec.split(":"))
    qd = torch.from_numpy(q[:nq]).cuda()
    for per in a.per.split(","):
        os.environ[a.env] = per
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
        balg = statistics.median(t["scanned_bytes"] for t in ts)
        print(json.dumps({"nq": nq, "nprobe": nprobe, a.env: int(per), "scan_ms": round(scan, 4),
                          "work_items": statistics.median(t["work_items"] for t in ts),
                          "alg_frac": round(balg / (scan / 1e3) / 1e9 / hbm, 3)}), flush=True)
    os.environ.pop(a.env, None)
