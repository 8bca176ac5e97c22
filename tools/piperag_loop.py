"""Config E (BASELINE.json configs[4]): PipeRAG's pipelined loop on one B200.

Retrieval (query-window embedding on the GPU + IVF-PQ search, batch 1,
k=2) on a high-priority side stream, overlapped with a synthetic RETRO-style
decode on the main stream (582M fp32 params streamed per token + KV cache),
1024 tokens, retrieval interval m' in {64, 32, 16}; modes retro (blocking,
non-stale query window) and piperag (pipelined, query window stale by one
interval), piperag with and without an SM partition (decode pinned to S - R
SMs, search grids on R); nprobe fixed (16) and auto (select_nprobe on the
GPU-calibrated retrieval model with the budget from the calibrated inference
model). Prints one JSON document.
  python tools/piperag_loop.py [--small] [--tokens 1024] [--rsms 0,8,16]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402
from paper_2403_05676_b200 import pipeline as PL  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--small", action="store_true")
ap.add_argument("--tokens", type=int, default=1024)
ap.add_argument("--params", type=int, default=582_000_000)
ap.add_argument("--rsms", default="0,8,16", help="retrieval SM budgets for piperag (0: no partition)")
ap.add_argument("--intervals", default="64,32,16")
a = ap.parse_args()
n, nlist = (1_000_000, 1024) if a.small else (10_000_000, 4096)
path, q, meta = F.ensure_fixture(n, 384, nlist, 32, 1, nq=64, log=lambda *x: print(*x, file=sys.stderr))
ix = pg.GpuIndex.load(path, 0)
qd = torch.from_numpy(q).cuda()
dec = PL.SyntheticDecoder(params=a.params, max_positions=a.tokens + 128)
# the token sequence: a 64-token prompt chunk then the generated tokens
# (synthetic ids in [1, 256]); the query windows are embedded on the GPU
gen = torch.Generator().manual_seed(7)
tokens = torch.randint(1, 257, (64 + a.tokens,), generator=gen, dtype=torch.int32).cuda()
emb = pg.GpuChunkEmbedder(384, seed=11, vocab=257)
for _ in range(3):  # warm both sides
    dec.generate_chunk(64, 4)
    ix.search_batch(qd[:1], 2, 16)
torch.cuda.synchronize()
imodels = {mp: PL.calibrate_inference(lambda p, mp=mp: dec.time_chunk(p, mp), [64, 256, 512, 1024], mp,
                                      repeats=3, warmups=1) for mp in [int(x) for x in a.intervals.split(",")]}
rmodel, lat = pg.calibrate_gpu(ix, q[:1], 2, [1, 2, 4, 8, 16, 32, 64, 128], repeats=5, warmups=2)
out = {"workload": f"PipeRAG loop: {a.tokens} tokens, decode stand-in {a.params / 1e6:.0f}M fp32 params "
                   f"({dec.bytes_per_token(0) / 1e9:.2f} GB/token) + KV cache; retrieval batch 1, k=2, "
                   f"IVF-PQ {n // 1_000_000}M x 384, nlist={nlist}, m=32",
       "retrieval_model": {"slope_s": rmodel.slope_s, "intercept_s": rmodel.intercept_s,
                           "fit_residual_s": rmodel.fit_residual_s, "latency_s": lat},
       "inference_model": {str(mp): [[b.position, b.seconds] for b in m.buckets] for mp, m in imodels.items()},
       "runs": []}
intervals = [int(x) for x in a.intervals.split(",")]
for mp in intervals:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dec.stream)  # decode only: the generation-time floor
    for j in range(1, a.tokens // mp + 1):
        dec.generate_chunk(64 + (j - 1) * mp, mp)
    e1.record(dec.stream)
    e1.synchronize()
    base = e0.elapsed_time(e1) / 1e3
    out["runs"].append({"interval": mp, "mode": "none", "total_latency_s": base})
    variants = [("retro", 0)] + [("piperag", int(r)) for r in a.rsms.split(",")]
    for mode, rs in variants:
        eng = PL.PipelineEngine(dec, ix, None, k=2, retrieval_model=rmodel, inference_model=imodels[mp],
                                embedder=emb, tokens=tokens, retrieval_sms=rs or None)
        for npb in (16, None):
            eng.run(mode, a.tokens, mp, nprobe=npb)  # warm
            tr = eng.run(mode, a.tokens, mp, nprobe=npb)
            rets = sorted(tr.durations("ret_start").values())
            out["runs"].append({
                "interval": mp, "mode": mode, "retrieval_sms": rs or "all (no partition)",
                "nprobe": "auto" if npb is None else npb,
                "total_latency_s": tr.total_latency_s, "stall_time_s": tr.stall_time_s,
                "stall_count": tr.stall_count, "retrievals": tr.retrieval_count,
                "nprobe_used_min": min(tr.nprobe_used), "nprobe_used_max": max(tr.nprobe_used),
                "retrieval_s_median": rets[len(rets) // 2],
                "overhead_vs_decode_only": tr.total_latency_s / base - 1.0})
print(json.dumps(out, indent=1))
