"""Times the device index build (prag_gpu_train_index) at config-A/B scale
against the reference's train_index (1,006 s for 1M x 384,
nlist 1024, nsq 32 on one core) and checks it bit-exact against the C
restatement on a bounded case. Prints one JSON line per case.

usage: python tools/train_bench.py [--n 1000000] [--d 384] [--nlist 1024] [--nsq 32] [--ref-n 20000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--d", type=int, default=384)
    ap.add_argument("--nlist", type=int, default=1024)
    ap.add_argument("--nsq", type=int, default=32)
    ap.add_argument("--ref-n", type=int, default=20000)
    ap.add_argument("--ref-nlist", type=int, default=128)
    a = ap.parse_args()
    import torch
    import _oracle as O
    import paper_2403_05676_b200 as pg

    # bounded exactness + CPU timing of the restatement (same algorithm)
    v = O.random_vectors(a.ref_n, a.d, 5)
    p = pg.TrainParams(nlist=a.ref_nlist, n_subquantizers=a.nsq)
    t0 = time.time()
    g = pg.train_index(v, p)
    t_gpu_small = time.time() - t0
    t0 = time.time()
    r = O.train_index(v, a.ref_nlist, a.nsq)
    t_cpu_small = time.time() - t0
    same = all((x.view(np.uint8) == y.view(np.uint8)).all() for x, y in
               zip((g.centroids, g.codewords, g.list_off, g.ids, g.codes), r))
    print(json.dumps({"case": f"{a.ref_n}x{a.d} nlist={a.ref_nlist} nsq={a.nsq}", "bit_exact_vs_oracle": bool(same),
                      "gpu_s": round(t_gpu_small, 3), "oracle_cpu_s_1core": round(t_cpu_small, 2)}), flush=True)

    # config-A-scale build: vectors generated on the device (N(0,1), torch RNG)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    x = torch.randn(a.n, a.d, generator=gen, device="cuda", dtype=torch.float32)
    p = pg.TrainParams(nlist=a.nlist, n_subquantizers=a.nsq)
    pg.train_index(x[:50_000], pg.TrainParams(nlist=64, n_subquantizers=a.nsq, kmeans_iterations=1))  # warm-up
    torch.cuda.synchronize()
    t0 = time.time()
    t = pg.train_index(x, p)
    torch.cuda.synchronize()
    el = time.time() - t0
    sizes = np.diff(t.list_off.astype(np.int64))
    print(json.dumps({"case": f"{a.n}x{a.d} nlist={a.nlist} nsq={a.nsq} (reference TrainParams defaults)",
                      "gpu_s": round(el, 3), "reference_s_published_in_survey": 1006.0 if a.n == 1_000_000 else None,
                      "list_p50": int(np.median(sizes)), "list_max": int(sizes.max())}), flush=True)


if __name__ == "__main__":
    main()
