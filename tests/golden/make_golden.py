"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs /root/reference): it builds
oracle/_ref/ref_tool from the unmodified reference headers (oracle/Makefile),
trains indexes with the reference prag::train_index, writes them with
prag::store_index, and records prag::search outputs. Committed outputs:

  <case>.pragix          PRAGIX01 index (annindex.hpp:335-359)
  <case>.npz             queries + per (nprobe, k) reference results

Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import _oracle as O  # noqa: E402


def two_clusters(per_cluster: int, d: int, seed: int) -> np.ndarray:
    """test_annindex.cpp:22-35."""
    rng = O.SplitMix64(seed)
    out = []
    for c in range(2):
        for _ in range(per_cluster):
            x = np.array([np.float32(np.float32(0.05) * np.float32(rng.next_gaussian()))
                          for _ in range(d)], dtype=np.float32)
            x[0] = np.float32(x[0] + np.float32(-10.0 if c == 0 else 10.0))
            out.append(x)
    return np.stack(out)


def train(tmp, name, vecs, nlist, nsq, seed=7):
    vpath = os.path.join(tmp, name + ".f32")
    vecs.astype(np.float32).tofile(vpath)
    out = os.path.join(HERE, name + ".pragix")
    O.ref_run("train", vpath, vecs.shape[0], vecs.shape[1], nlist, nsq, seed, out)
    return out


def record(tmp, name, index_path, queries, grid):
    qpath = os.path.join(tmp, name + ".q.f32")
    queries.astype(np.float32).tofile(qpath)
    payload = {"queries": queries.astype(np.float32)}
    for nprobe, k in grid:
        rpath = os.path.join(tmp, f"{name}.{nprobe}.{k}.bin")
        O.ref_run("search", index_path, qpath, queries.shape[0], nprobe, k, rpath)
        ids, dist, count, scanned, lists = O.read_ref_results(rpath, queries.shape[0], k)
        key = f"p{nprobe}_k{k}"
        payload[key + "_ids"] = ids
        payload[key + "_dist"] = dist
        payload[key + "_count"] = count
        payload[key + "_scanned"] = scanned
        payload[key + "_lists"] = lists
    payload["grid"] = np.array(grid, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **payload)
    print(f"{name}: {len(grid)} searches x {queries.shape[0]} queries")


def main():
    O.build_oracle()
    if not O.ref_available():
        sys.exit("oracle/_ref/ref_tool missing: needs /root/reference")
    with tempfile.TemporaryDirectory() as tmp:
        # test_annindex.cpp:60-71 four separated points, nlist 4, nsq 2.
        v = np.array([[0, 0], [10, 0], [0, 10], [10, 10]], dtype=np.float32)
        p = train(tmp, "four_points", v, 4, 2)
        record(tmp, "four_points", p, v, [(4, 1), (1, 4), (2, 10), (4, 4)])

        # test_annindex.cpp:127-143 two far clusters, nlist 2, nsq 4.
        v = two_clusters(100, 8, 5)
        p = train(tmp, "two_clusters", v, 2, 4)
        q = np.zeros((3, 8), dtype=np.float32)
        q[0, 0] = -10.0
        q[1, 0] = 10.0
        q[2, 1] = 3.0
        record(tmp, "two_clusters", p, q, [(1, 5), (2, 5), (2, 1000), (1, 1)])

        # test_annindex.cpp:145-163 data (600 x 16, nlist 16, nsq d/4) and its
        # query recipe (SplitMix64(60), +0.1 N(0,1)).
        v = O.random_vectors(600, 16, 6)
        p = train(tmp, "rand600_d16", v, 16, 0)
        q = O.noisy_queries(v, 30, 60, 0.1)
        record(tmp, "rand600_d16", p, q, [(1, 1), (1, 5), (4, 5), (16, 5), (16, 10), (3, 64)])

        # d=384 shapes with the hot-path PQ widths (m=32 / m=64): the layouts
        # the specialised scan kernels handle. Queries: annindex_main.cpp:66-74.
        v = O.random_vectors(2500, 384, 11)
        p = train(tmp, "d384_m32", v, 32, 32)
        q = O.noisy_queries(v, 40, 13, 0.05)
        record(tmp, "d384_m32", p, q, [(1, 1), (1, 10), (4, 10), (8, 10), (32, 10), (8, 100), (2, 2)])

        v = O.random_vectors(2500, 384, 12)
        p = train(tmp, "d384_m64", v, 32, 64)
        q = O.noisy_queries(v, 40, 13, 0.05)
        record(tmp, "d384_m64", p, q, [(1, 1), (1, 10), (4, 10), (8, 10), (32, 10), (8, 100)])

        v = O.random_vectors(3000, 64, 13)
        p = train(tmp, "d64_m16", v, 24, 16)
        q = O.noisy_queries(v, 32, 14, 0.05)
        record(tmp, "d64_m16", p, q, [(1, 10), (5, 10), (24, 10), (24, 257)])

        # Exact-tie fixture (hand-built index): integer codewords make many
        # candidate distances exactly equal, so the (distance, chunk_id)
        # tie-break of annindex.hpp:55-58 decides membership at the k-th place.
        # Lists 1, 4 and 6 are empty (annindex.hpp:290 skip path).
        rng = O.SplitMix64(99)
        nlist, d, nsq = 8, 8, 2
        cents = np.array([[float((l * 3 + j) % 5) for j in range(d)] for l in range(nlist)],
                         dtype=np.float32)
        words = np.zeros((nsq, 256, d // nsq), dtype=np.float32)
        for s in range(nsq):
            for c in range(256):
                for j in range(d // nsq):
                    words[s, c, j] = float((c * (j + 1) + s) % 3)
        perm = np.arange(400, dtype=np.uint64)
        for i in range(399, 0, -1):  # Fisher-Yates with SplitMix64
            j = rng.next_below(i + 1)
            perm[i], perm[j] = perm[j], perm[i]
        sizes = [70, 0, 120, 50, 0, 90, 0, 70]
        lists, at = [], 0
        for sz in sizes:
            ids = perm[at:at + sz]
            codes = np.array([[rng.next_below(6) for _ in range(nsq)] for _ in range(sz)],
                             dtype=np.uint8).reshape(sz, nsq)
            lists.append((ids, codes))
            at += sz
        p = os.path.join(HERE, "ties_empty.pragix")
        O.write_pragix(p, cents, words, lists)
        q = np.array([[float((i * 7 + j) % 4) * 0.5 for j in range(d)] for i in range(12)],
                     dtype=np.float32)
        record(tmp, "ties_empty", p, q,
               [(1, 1), (1, 7), (2, 13), (3, 50), (8, 1), (8, 33), (8, 400), (8, 1000), (5, 64)])


if __name__ == "__main__":
    main()
