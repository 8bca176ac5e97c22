"""Batch-1 device time per search: N back-to-back searches of one query on
device buffers (queued without host sync, so launch overhead overlaps), the
batch-1 kernel vs the five-kernel chain (default), config B.
  python tools/b1_time.py [--n 200]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200)
ap.add_argument("--k", type=int, default=2)
a = ap.parse_args()
path, q, _ = F.ensure_fixture(10_000_000, 384, 4096, 32, 1, nq=64, log=lambda *x: None)
ix = pg.GpuIndex.load(path, 0)
s = torch.cuda.Stream()
qd = torch.from_numpy(q[:1].copy()).cuda()
k = a.k
out = pg.BatchResult(torch.empty((1, k), dtype=torch.int64, device="cuda"),
                     torch.empty((1, k), dtype=torch.float32, device="cuda"),
                     torch.empty((1,), dtype=torch.int32, device="cuda"), torch.empty((1,), dtype=torch.int64, device="cuda"))
for mode in ("batch1", "chain"):
    os.environ["PRAG_GPU_BATCH1"] = "1" if mode == "batch1" else "0"
    for nprobe in (1, 16, 64):
        for _ in range(20):
            ix.search_batch(qd, k, nprobe, stream=s, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.n):
            ix.search_batch(qd, k, nprobe, stream=s, out=out)
        e1.record(s)
        e1.synchronize()
        print(json.dumps({"mode": mode, "nprobe": nprobe, "k": k, "us_per_search": round(e0.elapsed_time(e1) * 1e3 / a.n, 2)}), flush=True)
os.environ.pop("PRAG_GPU_BATCH1", None)
