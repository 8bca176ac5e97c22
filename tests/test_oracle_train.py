"""The oracle's C restatement of prag::train_index (oracle/prag_oracle.c,
ora_train_index) against the reference-written golden indexes
(tests/golden/*.pragix, tests/golden/train_cases.json): pins the restatement
that tests/test_gpu_train.py can fall back on for sizes without a golden file."""
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))

CASES = json.load(open(os.path.join(HERE, "golden", "train_cases.json")))


@pytest.mark.parametrize("case", CASES["cases"], ids=[c["name"] for c in CASES["cases"]])
def test_oracle_train_matches_reference_golden(case):
    import _oracle as O
    import make_train_golden as M
    from paper_2403_05676_b200.fixtures import read_pragix
    p = {**CASES["default"], **{k: case[k] for k in ("seed", "iters", "cap") if k in case}}
    got = O.train_index(M.vectors(case["gen"]), case["nlist"], case["nsq"], p["seed"], p["iters"], p["cap"])
    ref = read_pragix(os.path.join(HERE, "golden", case["name"] + ".pragix"))
    for name, a, b in zip(("centroids", "codewords", "list_off", "ids", "codes"), got, ref):
        assert a.shape == b.shape, name
        if a.dtype == np.float32:
            assert (a.view(np.uint32) == b.view(np.uint32)).all(), name
        else:
            assert (a == b).all(), name


def test_oracle_train_errors():
    import _oracle as O
    v = np.ones((10, 8), np.float32)
    for args, msg in [((v[:0], 2), "empty"), ((v, 11), "nlist exceeds"), ((v, 2, 3), "not divisible"),
                      ((v, 4, 0, 7, 25, 3), "fewer points")]:
        with pytest.raises(O.OracleError, match=msg):
            O.train_index(*args)
