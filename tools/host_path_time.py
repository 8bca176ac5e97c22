"""prag_gpu_search with host buffers (the drop-in call) per batch shape,
cached host plans on/off (PRAG_GPU_HOST_PLANS, read once per process: run
twice). Wall clock per call, p50 over --calls, config B.
  python tools/host_path_time.py"""
import argparse, json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--calls", type=int, default=200)
a = ap.parse_args()
path, q, _ = F.ensure_fixture(10_000_000, 384, 4096, 32, 1, nq=64, log=lambda *x: None)
ix = pg.GpuIndex.load(path, 0)
s = torch.cuda.Stream()
rows = []
for nq, k, nprobe in ((64, 10, 16), (16, 10, 16), (1, 2, 16), (1, 2, 1), (1, 2, 128)):
    qh = torch.from_numpy(q[:nq].copy()).pin_memory().numpy()
    out = pg.BatchResult(torch.empty((nq, k), dtype=torch.int64).pin_memory().numpy().view(np.uint64),
                         torch.empty((nq, k), dtype=torch.float32).pin_memory().numpy(),
                         torch.empty((nq,), dtype=torch.int32).pin_memory().numpy().view(np.uint32),
                         torch.empty((nq,), dtype=torch.int64).pin_memory().numpy().view(np.uint64))
    for _ in range(10):
        ix.search_batch(qh, k, nprobe, stream=s, out=out)
    ts = []
    for _ in range(a.calls):
        t0 = time.perf_counter()
        ix.search_batch(qh, k, nprobe, stream=s, out=out)
        ts.append((time.perf_counter() - t0) * 1e6)
    rows.append({"nq": nq, "k": k, "nprobe": nprobe, "us_p50": round(statistics.median(ts), 1),
                 "qps": round(nq / statistics.median(ts) * 1e6, 1)})
print(json.dumps({"host_plans": os.environ.get("PRAG_GPU_HOST_PLANS", "1"), "rows": rows}))
