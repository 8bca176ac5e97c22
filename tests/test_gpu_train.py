"""Device index build (prag_gpu_train_index) == the reference's
prag::train_index (annindex.hpp:164-241), bit for bit: centroids, codewords,
list membership and order, ids and codes are compared with the PRAGIX01 files
the reference itself wrote (tests/golden/*.pragix; make_golden.py and
make_train_golden.py). The mirrors the reference's own build tests
(test_annindex.cpp: every vector assigned exactly once, round trip through
store/load, validation errors)."""
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))

pytestmark = pytest.mark.gpu

CASES = json.load(open(os.path.join(HERE, "golden", "train_cases.json")))


def _params(case):
    import paper_2403_05676_b200 as pg
    d = {**CASES["default"], **{k: case[k] for k in ("seed", "iters", "cap") if k in case}}
    return pg.TrainParams(nlist=case["nlist"], n_subquantizers=case["nsq"], seed=d["seed"],
                          kmeans_iterations=d["iters"], train_sample_cap=d["cap"])


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    if a.dtype == np.float32:
        return (a.view(np.uint32) == b.view(np.uint32)).all()
    return (a == b).all()


@pytest.mark.parametrize("case", CASES["cases"], ids=[c["name"] for c in CASES["cases"]])
def test_train_matches_reference_golden(case, tmp_path):
    import make_train_golden as M
    import paper_2403_05676_b200 as pg
    from paper_2403_05676_b200.fixtures import read_pragix
    v = M.vectors(case["gen"])
    t = pg.train_index(v, _params(case))
    gc, gw, go, gi, gk = read_pragix(os.path.join(HERE, "golden", case["name"] + ".pragix"))
    assert _same(t.centroids, gc), "centroids differ"
    assert _same(t.codewords, gw), "codewords differ"
    assert _same(t.list_off, go), "list sizes differ"
    assert _same(t.ids, gi), "list membership / order differ"
    assert _same(t.codes, gk), "codes differ"
    # store_index byte-identity (annindex.hpp:335-359)
    out = tmp_path / "x.pragix"
    t.write_pragix(str(out))
    assert out.read_bytes() == open(os.path.join(HERE, "golden", case["name"] + ".pragix"), "rb").read()


def test_train_every_vector_assigned_once_and_searchable():
    """test_annindex.cpp:73-100 spirit: each vector in exactly one list; the
    trained index serves searches identical to the oracle's on the same file."""
    import _oracle as O
    import paper_2403_05676_b200 as pg
    v = O.random_vectors(4000, 64, 41)
    t = pg.train_index(v, pg.TrainParams(nlist=32, n_subquantizers=16))
    assert int(t.list_off[-1]) == 4000
    assert np.array_equal(np.sort(t.ids), np.arange(4000, dtype=np.uint64))
    for l in range(32):
        seg = t.ids[int(t.list_off[l]):int(t.list_off[l + 1])]
        assert (np.diff(seg.astype(np.int64)) > 0).all()  # vector order inside a list
    ix = t.to_gpu()
    q = O.noisy_queries(v, 16, 3, 0.05)
    r = ix.search_batch(q, 10, 8)
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        p = os.path.join(tmp, "t.pragix")
        t.write_pragix(p)
        ids, dist, count, scanned = O.OracleIndex(p).search(q, 8, 10)[:4]
    assert (r.ids == ids).all() and (r.dist.view(np.uint32) == dist.view(np.uint32)).all()
    assert (r.count == count).all() and (r.scanned == scanned).all()


def test_train_device_input_same_as_host():
    import torch
    import _oracle as O
    import paper_2403_05676_b200 as pg
    v = O.random_vectors(3000, 32, 42)
    p = pg.TrainParams(nlist=20, n_subquantizers=8, kmeans_iterations=5)
    a = pg.train_index(v, p)
    b = pg.train_index(torch.from_numpy(v).cuda(), p)
    for x, y in [(a.centroids, b.centroids), (a.codewords, b.codewords), (a.list_off, b.list_off),
                 (a.ids, b.ids), (a.codes, b.codes)]:
        assert _same(x, y)


def test_train_validation_errors():
    """annindex.hpp:166-174, :66 (test_annindex.cpp:176-192 style)."""
    import paper_2403_05676_b200 as pg
    v = np.random.default_rng(0).standard_normal((50, 8)).astype(np.float32)
    with pytest.raises(pg.ConfigError, match="empty embedding set"):
        pg.train_index(np.zeros((0, 8), np.float32), pg.TrainParams(nlist=4))
    with pytest.raises(pg.ConfigError, match="nlist exceeds number of vectors"):
        pg.train_index(v, pg.TrainParams(nlist=51))
    with pytest.raises(pg.ConfigError, match="not divisible"):
        pg.train_index(v, pg.TrainParams(nlist=4, n_subquantizers=3))
    with pytest.raises(pg.ConfigError, match="fewer points than clusters"):
        pg.train_index(v, pg.TrainParams(nlist=20, train_sample_cap=10))


def test_train_matches_oracle_larger():
    """Sample-capped, > 128 lists, d = 64: against the pinned C restatement
    (tests/test_oracle_train.py) at a size it trains in seconds."""
    import _oracle as O
    import paper_2403_05676_b200 as pg
    v = O.random_vectors(12000, 64, 43)
    t = pg.train_index(v, pg.TrainParams(nlist=160, n_subquantizers=16, kmeans_iterations=6, train_sample_cap=6000))
    ref = O.train_index(v, 160, 16, 7, 6, 6000)
    for x, y in zip((t.centroids, t.codewords, t.list_off, t.ids, t.codes), ref):
        assert _same(x, y)


@pytest.mark.parametrize("case", [c["name"] for c in CASES["cases"]][:6])
def test_store_roundtrip_is_byte_identical(case, tmp_path):
    """prag_gpu_index_store (annindex.hpp:335-359): load a reference-written
    PRAGIX01 into HBM, store it back: the same bytes."""
    import paper_2403_05676_b200 as pg
    src = os.path.join(HERE, "golden", case + ".pragix")
    ix = pg.GpuIndex.load(src)
    out = tmp_path / "back.pragix"
    ix.store(str(out))
    assert out.read_bytes() == open(src, "rb").read()
