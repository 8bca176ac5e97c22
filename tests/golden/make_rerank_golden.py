"""Golden outputs of the reference's search with exact_rerank = true
(annindex.hpp:307-312), made by oracle/_ref/ref_tool (the unmodified
reference headers) on the trained golden indexes whose input vectors are
regenerable (make_train_golden.EXISTING). Writes tests/golden/rerank.npz:
per case and (nprobe, k) the ids / dist / count / scanned arrays.

Usage: python tests/golden/make_rerank_golden.py
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
import _oracle as O  # noqa: E402
import make_train_golden as M  # noqa: E402

CASES = {"rand600_d16": [(1, 5), (4, 10), (16, 10)], "d384_m32": [(1, 10), (8, 10), (32, 10), (8, 100)],
         "d64_m16": [(5, 10), (24, 10), (24, 257)]}


def main():
    O.build_oracle()
    if not O.ref_available():
        sys.exit("oracle/_ref/ref_tool missing: needs /root/reference")
    gens = {c["name"]: c["gen"] for c in M.EXISTING}
    payload = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, grid in CASES.items():
            v = M.vectors(gens[name])
            q = np.load(os.path.join(HERE, name + ".npz"))["queries"]
            vp, qp = os.path.join(tmp, "v.f32"), os.path.join(tmp, "q.f32")
            v.tofile(vp)
            q.astype(np.float32).tofile(qp)
            for nprobe, k in grid:
                rp = os.path.join(tmp, "r.bin")
                O.ref_run("rerank", os.path.join(HERE, name + ".pragix"), vp, v.shape[0], qp, q.shape[0], nprobe, k,
                          rp)
                ids, dist, count, scanned, _ = O.read_ref_results(rp, q.shape[0], k)
                key = f"{name}_p{nprobe}_k{k}"
                payload[key + "_ids"], payload[key + "_dist"] = ids, dist
                payload[key + "_count"], payload[key + "_scanned"] = count, scanned
            print(name, grid)
    np.savez_compressed(os.path.join(HERE, "rerank.npz"), **payload)


if __name__ == "__main__":
    main()
