"""Phase timeline of the batch-1 kernel from a trace build (touch
csrc/batch1.cu; make -C paper_2403_05676_b200/csrc EXTRA=-DPRAG_B1_TRACE):
per CTA the globaltimer after setup (0), after the coarse slice (1), after
barrier 1 (2), after the probe selection (3), after the table rows (4),
after barrier 2 (5), after the scan (6), after the CTA merge (7), and the
final merge's end (8, last CTA only); microseconds from the earliest mark 0.
  python tools/b1_trace.py [--nprobe 16] [--k 2]"""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PRAG_GPU_BATCH1"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2403_05676_b200 as pg  # noqa: E402
from paper_2403_05676_b200 import fixtures as F  # noqa: E402
from paper_2403_05676_b200._lib import lib  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--nprobe", type=int, default=16)
ap.add_argument("--k", type=int, default=2)
a = ap.parse_args()
path, q, _ = F.ensure_fixture(10_000_000, 384, 4096, 32, 1, nq=64, log=lambda *x: None)
ix = pg.GpuIndex.load(path, 0)
qd = torch.from_numpy(q[:1].copy()).cuda()
f = lib().prag_gpu_debug_b1_trace
f.argtypes = [C.c_void_p, C.c_size_t]
out = []
for rep in range(6):
    ix.search_batch(qd, a.k, a.nprobe)
    torch.cuda.synchronize()
    buf = np.zeros(256 * 16, dtype=np.uint64)
    assert f(buf.ctypes.data, buf.size) == 0
    t = buf.reshape(256, 16)[:torch.cuda.get_device_properties(0).multi_processor_count].astype(np.int64)
    base = t[:, 0].min()
    row = {}
    for i in range(8):
        v = (t[:, i] - base) / 1e3
        row[i] = [round(float(v.min()), 2), round(float(np.median(v)), 2), round(float(v.max()), 2)]
    row[8] = round(float((t[:, 8].max() - base) / 1e3), 2)
    out.append(row)
print(json.dumps({"nprobe": a.nprobe, "k": a.k, "marks_min_med_max_us": out[-1], "end_us_per_rep": [r[8] for r in out]}))
