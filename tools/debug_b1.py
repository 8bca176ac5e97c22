"""Debug aid: batch-1 searches on one golden fixture, one call per line."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2403_05676_b200 as pg
from conftest import load_golden
case = sys.argv[1] if len(sys.argv) > 1 else "d384_m64"
path, z, grid = load_golden(case)
ix = pg.GpuIndex.load(path, 0)
q = z["queries"]
for nprobe, k in grid:
    if k > 32:
        continue
    for i in range(2):
        print("call", nprobe, k, i, flush=True)
        r = ix.search_batch(q[i:i + 1], k, nprobe)
        print(r.ids[0, :r.count[0]], flush=True)
