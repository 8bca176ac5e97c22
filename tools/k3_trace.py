"""K3 timeline from a trace build (make -C paper_2403_05676_b200/csrc
EXTRA=-DPRAG_K3_TRACE after touching scan_skew.cu): per CTA the time after
pdl_wait, each item consumer warp 0 scanned (start = image ready, end), and
the exit; summarised as start/finish spreads, per-item time and tiles/us, and
the gap between an item's end and the next image.
  python tools/k3_trace.py [--n ..] [--nlist ..] [--m ..] [--seed ..] --nq 1 --nprobe 128"""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402
from paper_2403_05676_b200._lib import lib  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--nlist", type=int, default=16384)
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--seed", type=int, default=3)
ap.add_argument("--nq", type=int, default=1)
ap.add_argument("--nprobe", type=int, default=128)
ap.add_argument("--tail", action="store_true", help="also print the last items of the last CTAs to finish")
a = ap.parse_args()
path, q, _ = F.ensure_fixture(a.n, 384, a.nlist, a.m, a.seed, nq=64, log=lambda *x: None)
ix = pg.GpuIndex.load(path, 0)
qd = torch.from_numpy(q[:a.nq]).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ix.search_batch(qd, 10, a.nprobe)
flush.zero_()
torch.cuda.synchronize()
ix.search_batch(qd, 10, a.nprobe)
torch.cuda.synchronize()
L = lib()
f = L.prag_gpu_debug_k3_trace
f.argtypes = [C.c_void_p, C.c_size_t]
buf = np.zeros(160 * 256, dtype=np.uint64)
assert f(buf.ctypes.data, buf.size) == 0
tr = buf.reshape(160, 256)
sms = torch.cuda.get_device_properties(0).multi_processor_count
ctas = []
for c in range(sms):
    row = tr[c]
    n = int(row[255])
    t0 = int(row[0])
    ev = [int(x) for x in row[1:n]]
    items = []
    end = None
    i = 0
    while i < len(ev):
        if ev[i] >> 63:
            end = ev[i] & ((1 << 63) - 1)
            i += 1
            continue
        items.append((ev[i], ev[i + 1], ev[i + 2]))
        i += 3
    ctas.append((t0, items, end))
base = min(c[0] for c in ctas)
starts = [(c[0] - base) / 1e3 for c in ctas]
ends = [((c[2] or c[1][-1][1]) - base) / 1e3 for c in ctas]
first_item = [((c[1][0][0] if c[1] else c[2]) - base) / 1e3 for c in ctas]
item_us = [(e - s) / 1e3 for c in ctas for (s, e, t) in c[1]]
rate = [t / max((e - s) / 1e3, 1e-9) for c in ctas for (s, e, t) in c[1]]
gaps = [(c[1][j + 1][0] - c[1][j][1]) / 1e3 for c in ctas for j in range(len(c[1]) - 1)]
busy = [sum((e - s) for (s, e, t) in c[1]) / 1e3 for c in ctas]
pct = lambda v, p: round(float(np.percentile(v, p)), 2) if v else None
print(json.dumps({
    "shape": {"n": a.n, "nlist": a.nlist, "m": a.m, "nq": a.nq, "nprobe": a.nprobe},
    "kernel_span_us": round(max(ends), 2),
    "cta_start_us": [pct(starts, 0), pct(starts, 50), pct(starts, 100)],
    "first_image_ready_us": [pct(first_item, 0), pct(first_item, 50), pct(first_item, 100)],
    "cta_finish_us": [pct(ends, 0), pct(ends, 10), pct(ends, 50), pct(ends, 90), pct(ends, 100)],
    "items_per_cta": [min(len(c[1]) for c in ctas), float(np.mean([len(c[1]) for c in ctas])), max(len(c[1]) for c in ctas)],
    "item_us": [pct(item_us, 10), pct(item_us, 50), pct(item_us, 90), pct(item_us, 100)],
    "tiles_per_us_warp0": [pct(rate, 10), pct(rate, 50), pct(rate, 90)],
    "gap_between_items_us": [pct(gaps, 50), pct(gaps, 90), pct(gaps, 100)] if gaps else None,
    "busy_frac_warp0": round(float(np.mean(busy)) / max(ends), 3),
}))
if a.tail:
    f2 = L.prag_gpu_debug_k3_trace2
    f2.argtypes = [C.c_void_p, C.c_size_t]
    b2 = np.zeros(160 * 6 * 32, dtype=np.uint64)
    assert f2(b2.ctypes.data, b2.size) == 0
    t2 = b2.reshape(160, 6, 32).astype(np.int64)
    # per-warp item ends: only builds that record them (prag_gpu_debug_k3_trace3)
    b3 = np.zeros(160 * 16 * 32, dtype=np.uint64)
    if hasattr(L, "prag_gpu_debug_k3_trace3"):
        f3 = L.prag_gpu_debug_k3_trace3
        f3.argtypes = [C.c_void_p, C.c_size_t]
        assert f3(b3.ctypes.data, b3.size) == 0
    t3 = b3.reshape(160, 16, 32).astype(np.int64)
    order = np.argsort(ends)
    lag = []  # per CTA and item: slowest consumer warp's range end minus the median warp's
    for c in range(sms):
        for j in range(len(ctas[c][1])):
            v = [int(t3[c, w, j]) for w in range(16) if t3[c, w, j]]
            if len(v) > 2:
                lag.append((max(v) - float(np.median(v))) / 1e3)
    print(json.dumps({"item_warp_lag_us_p50_p90_max": [pct(lag, 50), pct(lag, 90), pct(lag, 100)]}))
    for c in list(order[-2:]):
        n = len(ctas[c][1])
        print(json.dumps({"cta": int(c), "per_item_warp_end_us": [[round((int(t3[c, w, j]) - base) / 1e3, 1) if t3[c, w, j] else None for w in range(16)] for j in range(n)]}))
    for c in list(order[:2]) + list(order[-4:]):
        n = len(ctas[c][1])
        ev = [[round((int(t2[c, k, j]) - base) / 1e3, 2) if t2[c, k, j] else None for k in range(6)] for j in range(n)]
        print(json.dumps({"cta": int(c), "tiles": [int(t_) for (_, _, t_) in ctas[c][1]],
                          "per_item_fetched_staged_stgseen_buffree_imgready_lastwarpdone": ev}))
    for c in list(order[:3]) + list(order[-8:]):
        t0, items, end = ctas[c]
        print(json.dumps({"cta": int(c), "end": round(ends[c], 2), "n_items": len(items),
                          "last_items_start_end_tiles": [[round((s_ - base) / 1e3, 2), round((e_ - base) / 1e3, 2), int(t_)]
                                                         for (s_, e_, t_) in items[-6:]]}))
    allit = sorted(((s_ - base) / 1e3, t_) for c in ctas for (s_, e_, t_) in c[1])
    print(json.dumps({"items_total": len(allit), "tiles_total": int(sum(t for _, t in allit)),
                      "tiles_of_items_started_after_p50_finish": int(sum(t for s_, t in allit if s_ > pct(ends, 50))),
                      "items_started_after_p50_finish": int(sum(1 for s_, t in allit if s_ > pct(ends, 50))),
                      "last_30_items_tiles": [int(t) for _, t in allit[-30:]]}))
