"""Device-resident search step, captured plan vs direct (PDL-chained)
launches, timed like bench.py (L2 flushed, CUDA events around one step).
  python tools/plan_vs_direct.py"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402
path, q, _ = F.ensure_fixture(10_000_000, 384, 4096, 32, 1, nq=64, log=lambda *x: None)
ix = pg.GpuIndex.load(path, 0)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []
for nq, k, nprobe in ((64, 10, 16), (64, 10, 64), (16, 10, 16), (1, 2, 16)):
    qd = torch.from_numpy(q[:nq].copy()).cuda()
    out = pg.BatchResult(torch.empty((nq, k), dtype=torch.int64, device="cuda"),
                         torch.empty((nq, k), dtype=torch.float32, device="cuda"),
                         torch.empty((nq,), dtype=torch.int32, device="cuda"), torch.empty((nq,), dtype=torch.int64, device="cuda"))
    plan = ix.plan(qd, k, nprobe, out, stream=s)
    res = {}
    for mode in ("plan", "direct"):
        fn = (lambda: plan.launch(stream=s)) if mode == "plan" else (lambda: ix.search_batch(qd, k, nprobe, stream=s, out=out))
        ts = []
        for i in range(60):
            with torch.cuda.stream(s):
                flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            if i >= 10:
                ts.append(e0.elapsed_time(e1) * 1e3)
        res[mode] = round(statistics.median(ts), 1)
    rows.append({"nq": nq, "nprobe": nprobe, "k": k, "plan_us": res["plan"], "direct_us": res["direct"]})
print(json.dumps(rows))
