"""Exact rerank (SearchParams::exact_rerank, annindex.hpp:307-312) on the GPU:
prag_gpu_search_rerank against outputs the reference search() itself wrote
with exact_rerank = true (tests/golden/rerank.npz, make_rerank_golden.py), and
the reference acceptance property C1 (acceptance.cpp:67-87,
test_annindex.cpp:145-163): probing every list with rerank returns exactly the
brute-force top-k (oracle ora_brute_force, annindex.hpp:244-257)."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(HERE, "golden", "rerank.npz"))
CASES = sorted({k.rsplit("_p", 1)[0] for k in GOLD.files})


def _vectors(name):
    import make_train_golden as M
    gen = {c["name"]: c["gen"] for c in M.EXISTING}[name]
    return M.vectors(gen)


@pytest.mark.parametrize("name", CASES)
def test_rerank_matches_reference_golden(name):
    import paper_2403_05676_b200 as pg
    ix = pg.GpuIndex.load(os.path.join(HERE, "golden", name + ".pragix"))
    v = _vectors(name)
    ix.set_embeddings(v)
    q = np.load(os.path.join(HERE, "golden", name + ".npz"))["queries"]
    keys = sorted({k[len(name) + 1:].rsplit("_", 1)[0] for k in GOLD.files if k.startswith(name + "_p")})
    for key in keys:
        nprobe, k = (int(x[1:]) for x in key.split("_"))
        r = ix.search_batch(q, k, nprobe, exact_rerank=True)
        g = {f: GOLD[f"{name}_{key}_{f}"] for f in ("ids", "dist", "count", "scanned")}
        assert (r.count == g["count"]).all() and (r.scanned == g["scanned"]).all(), key
        for i in range(q.shape[0]):
            c = int(g["count"][i])
            assert (r.ids[i, :c] == g["ids"][i, :c]).all(), (key, i)
            assert (r.dist[i, :c].view(np.uint32) == g["dist"][i, :c].view(np.uint32)).all(), (key, i)


def test_full_probe_rerank_equals_brute_force():
    """C1: nprobe = nlist with rerank is exact k-NN (ties by lower id)."""
    import _oracle as O
    import paper_2403_05676_b200 as pg
    name = "d64_m16"
    ix = pg.GpuIndex.load(os.path.join(HERE, "golden", name + ".pragix"))
    v = _vectors(name)
    ix.set_embeddings(v)
    q = np.load(os.path.join(HERE, "golden", name + ".npz"))["queries"]
    for k in (1, 10, 50):
        r = ix.search_batch(q, k, ix.nlist, exact_rerank=True)
        for i in range(q.shape[0]):
            ids = np.zeros(k, np.uint64)
            dist = np.zeros(k, np.float32)
            cnt = np.zeros(1, np.uint32)
            assert O.lib().ora_brute_force(O._p(v), v.shape[0], v.shape[1], O._p(q[i]), k, O._p(ids), O._p(dist),
                                           O._p(cnt)) == 0
            c = int(cnt[0])
            assert int(r.count[i]) == c
            assert (r.ids[i, :c] == ids[:c]).all()
            assert (r.dist[i, :c].view(np.uint32) == dist[:c].view(np.uint32)).all()


def test_rerank_errors_and_python_mirror():
    import paper_2403_05676_b200 as pg
    name = "rand600_d16"
    ix = pg.GpuIndex.load(os.path.join(HERE, "golden", name + ".pragix"))
    q = np.load(os.path.join(HERE, "golden", name + ".npz"))["queries"]
    with pytest.raises(pg.ConfigError, match="exact_rerank requires raw embeddings"):
        ix.search_batch(q, 5, 4, exact_rerank=True)
    with pytest.raises(pg.ConfigError, match="exact_rerank requires raw embeddings"):
        pg.search(ix, q[0], pg.SearchParams(nprobe=4, k=5, exact_rerank=True))
    v = _vectors(name)
    with pytest.raises(pg.ConfigError, match="no embedding row"):
        ix.set_embeddings(v[:100])
    r = pg.search(ix, q[0], pg.SearchParams(nprobe=4, k=5, exact_rerank=True), embeddings=v)
    g_ids = GOLD[f"{name}_p4_k10_ids"][0][:5]
    assert [n.chunk_id for n in r.neighbors] == [int(x) for x in g_ids]
