"""The CPU oracle (oracle/prag_oracle.c) is pinned to the reference itself:
golden fixtures in tests/golden/ were produced by the unmodified reference
(oracle/_ref/ref_tool, built from /root/reference by oracle/Makefile)."""
import numpy as np
import pytest

import _oracle as O
from conftest import GOLDEN_CASES, load_golden


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_oracle_matches_reference_golden(case):
    path, z, grid = load_golden(case)
    idx = O.OracleIndex(path)
    q = z["queries"]
    for nprobe, k in grid:
        key = f"p{nprobe}_k{k}"
        ids, dist, count, scanned = idx.search(q, nprobe, k)
        np.testing.assert_array_equal(count, z[key + "_count"], err_msg=key)
        np.testing.assert_array_equal(scanned, z[key + "_scanned"], err_msg=key)
        for i in range(q.shape[0]):
            c = count[i]
            np.testing.assert_array_equal(ids[i, :c], z[key + "_ids"][i, :c], err_msg=key)
            # bit-exact distances
            np.testing.assert_array_equal(dist[i, :c].view(np.uint32),
                                          z[key + "_dist"][i, :c].view(np.uint32), err_msg=key)
        assert (z[key + "_lists"] == nprobe).all()


def test_golden_ties_are_exercised():
    """The tie fixture must have equal distances straddling the k-th place."""
    path, z, grid = load_golden("ties_empty")
    hits = 0
    for nprobe, k in grid:
        key = f"p{nprobe}_k{k}"
        d = z[key + "_dist"]
        c = z[key + "_count"]
        for i in range(d.shape[0]):
            row = d[i, :c[i]]
            if len(row) > 1 and (np.diff(row) == 0).any():
                hits += 1
    assert hits > 10


def test_tie_break_kat():
    """test_annindex.cpp:50-58: {1,0},{0,1},{1,0},{0,1} vs {1,0} -> 0,2,1,3."""
    vecs = np.array([[1, 0], [0, 1], [1, 0], [0, 1]], dtype=np.float32)
    q = np.array([1, 0], dtype=np.float32)
    ids = np.zeros(4, dtype=np.uint64)
    dist = np.zeros(4, dtype=np.float32)
    cnt = np.zeros(1, dtype=np.uint32)
    O.lib().ora_brute_force(O._p(vecs), 4, 2, O._p(q), 4, O._p(ids), O._p(dist), O._p(cnt))
    assert list(ids) == [0, 2, 1, 3]


def test_validation_errors():
    path, z, grid = load_golden("rand600_d16")
    idx = O.OracleIndex(path)
    q = z["queries"][:1]
    for nprobe, k in [(0, 1), (idx.nlist + 1, 1), (1, 0)]:
        with pytest.raises(O.OracleError) as e:
            idx.search(q, nprobe, k)
        assert e.value.code == 1


def test_load_errors(tmp_path):
    with pytest.raises(O.OracleError) as e:
        O.OracleIndex(str(tmp_path / "missing.bin"))
    assert e.value.code == 2 and "cannot open" in str(e.value)
    p = tmp_path / "bad.bin"
    p.write_bytes(b"NOTMAGIC" + b"\0" * 40)
    with pytest.raises(O.OracleError) as e:
        O.OracleIndex(str(p))
    assert "bad index magic at offset 0" in str(e.value)
    src = open(load_golden("rand600_d16")[0], "rb").read()
    p.write_bytes(src[:-3])
    with pytest.raises(O.OracleError) as e:
        O.OracleIndex(str(p))
    assert "truncated posting code at offset" in str(e.value)


def test_select_nprobe_kats():
    """test_perfmodel.cpp:54-68."""
    s, b = 0.5e-3, 2e-3
    assert O.select_nprobe(s, b, 10e-3, 1024, 0.0) == 16
    assert O.select_nprobe(s, b, 10e-3, 1024) == 14
    assert O.select_nprobe(s, b, 10e-3, 8, 0.0) == 8
    assert O.select_nprobe(s, b, 1e-3, 1024) == 1
    assert O.select_nprobe(s, b, 0.0, 1024) == 1
    assert O.select_nprobe(0.0, 2e-3, 10e-3, 64) == 64


def test_least_squares_exact_line():
    """test_perfmodel.cpp:11-19 / :167-177."""
    x = np.array([1, 2, 4, 8, 16, 32], dtype=np.float64)
    y = 2e-3 + 0.5e-3 * x
    slope, icpt, res, r2 = O.least_squares(x, y)
    assert abs(slope - 0.5e-3) < 1e-9 and abs(icpt - 2e-3) < 1e-9 and res < 1e-9
    assert r2 == pytest.approx(1.0)
