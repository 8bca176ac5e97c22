"""Golden fixtures for the device index build (prag_gpu_train_index), made by
the REFERENCE's own prag::train_index + prag::store_index (oracle/_ref/ref_tool,
compiled from the unmodified headers).

Besides the trained golden indexes make_golden.py already holds (listed in
EXISTING with the inputs that made them), this adds cases that reach every
branch of annindex.hpp:62-241: the training sample (n > cap, :134-145,
:178-180), duplicate points (kmeans++ total == 0 -> next_below, :92-94; empty
clusters re-seeded from the farthest point, :119-126), zero Lloyd iterations,
fewer vectors than 256 PQ codes (:209), a sample smaller than 256 (codes past
the trained clusters stay zero but are still candidates in encoding, :217 and
:229), more than 128 lists, a non-default seed.

Inputs are regenerated bit-exactly from their recipe (SplitMix64 through the
oracle's C restatement), so only the PRAGIX01 outputs and train_cases.json are
committed.

Usage: python tests/golden/make_train_golden.py
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import _oracle as O  # noqa: E402

DEFAULT = {"seed": 7, "iters": 25, "cap": 32768}

# already committed by make_golden.py (reference-trained with the defaults)
EXISTING = [
    {"name": "four_points", "gen": {"kind": "four_points"}, "nlist": 4, "nsq": 2},
    {"name": "two_clusters", "gen": {"kind": "two_clusters", "per": 100, "d": 8, "seed": 5}, "nlist": 2, "nsq": 4},
    {"name": "rand600_d16", "gen": {"kind": "random", "n": 600, "d": 16, "seed": 6}, "nlist": 16, "nsq": 0},
    {"name": "d384_m32", "gen": {"kind": "random", "n": 2500, "d": 384, "seed": 11}, "nlist": 32, "nsq": 32},
    {"name": "d384_m64", "gen": {"kind": "random", "n": 2500, "d": 384, "seed": 12}, "nlist": 32, "nsq": 64},
    {"name": "d64_m16", "gen": {"kind": "random", "n": 3000, "d": 64, "seed": 13}, "nlist": 24, "nsq": 16},
]

NEW = [
    {"name": "train_cap", "gen": {"kind": "random", "n": 5000, "d": 48, "seed": 21}, "nlist": 40, "nsq": 12,
     "cap": 2048},
    {"name": "train_dups", "gen": {"kind": "dups", "k": 9, "n": 700, "d": 8, "seed": 22}, "nlist": 16, "nsq": 4},
    {"name": "train_iters0", "gen": {"kind": "random", "n": 1000, "d": 16, "seed": 23}, "nlist": 8, "nsq": 4,
     "iters": 0},
    {"name": "train_small_n", "gen": {"kind": "random", "n": 100, "d": 8, "seed": 24}, "nlist": 4, "nsq": 2},
    {"name": "train_cap_small", "gen": {"kind": "random", "n": 1000, "d": 8, "seed": 25}, "nlist": 4, "nsq": 4,
     "cap": 200},
    {"name": "train_seed", "gen": {"kind": "random", "n": 3000, "d": 32, "seed": 26}, "nlist": 50, "nsq": 8,
     "seed": 12345, "iters": 7},
    {"name": "train_nlist300", "gen": {"kind": "random", "n": 8000, "d": 32, "seed": 27}, "nlist": 300, "nsq": 8,
     "iters": 10},
]


def two_clusters(per_cluster: int, d: int, seed: int) -> np.ndarray:
    """test_annindex.cpp:22-35 (same recipe as make_golden.two_clusters)."""
    rng = O.SplitMix64(seed)
    out = []
    for c in range(2):
        for _ in range(per_cluster):
            x = np.array([np.float32(np.float32(0.05) * np.float32(rng.next_gaussian()))
                          for _ in range(d)], dtype=np.float32)
            x[0] = np.float32(x[0] + np.float32(-10.0 if c == 0 else 10.0))
            out.append(x)
    return np.stack(out)


def vectors(gen: dict) -> np.ndarray:
    k = gen["kind"]
    if k == "four_points":
        return np.array([[0, 0], [10, 0], [0, 10], [10, 10]], dtype=np.float32)
    if k == "two_clusters":
        return two_clusters(gen["per"], gen["d"], gen["seed"])
    if k == "random":
        return O.random_vectors(gen["n"], gen["d"], gen["seed"])
    if k == "dups":
        base = O.random_vectors(gen["k"], gen["d"], gen["seed"])
        rng = O.SplitMix64(gen["seed"] + 1)
        return np.stack([base[rng.next_below(gen["k"])] for _ in range(gen["n"])]).astype(np.float32)
    raise ValueError(k)


def params(case: dict) -> dict:
    return {**DEFAULT, **{k: case[k] for k in ("seed", "iters", "cap") if k in case}}


def main():
    O.build_oracle()
    if not O.ref_available():
        sys.exit("oracle/_ref/ref_tool missing: needs /root/reference")
    with tempfile.TemporaryDirectory() as tmp:
        for case in NEW:
            v = vectors(case["gen"])
            p = params(case)
            vpath = os.path.join(tmp, case["name"] + ".f32")
            v.astype(np.float32).tofile(vpath)
            out = os.path.join(HERE, case["name"] + ".pragix")
            O.ref_run("train", vpath, v.shape[0], v.shape[1], case["nlist"], case["nsq"], p["seed"], out,
                      p["iters"], p["cap"])
            print(f"{case['name']}: n={v.shape[0]} d={v.shape[1]} {p}")
    with open(os.path.join(HERE, "train_cases.json"), "w") as f:
        json.dump({"default": DEFAULT, "cases": EXISTING + NEW}, f, indent=1)


if __name__ == "__main__":
    main()
