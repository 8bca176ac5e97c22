"""GPU parity: the sm_100a search path through the C ABI against
(1) the reference's own outputs (tests/golden, produced by the unmodified
reference) and (2) the CPU oracle on larger seeded fixtures. Bar: ids
bit-exact in (distance, id) order, distances bit-exact (stricter than the
north star's 1e-5 relative), count and scanned_vectors equal."""
import os
import threading

import numpy as np
import pytest

import _oracle as O
from conftest import GOLDEN_CASES, load_golden

pg = pytest.importorskip("paper_2403_05676_b200")
pytestmark = pytest.mark.gpu

MAXREL = 1e-5  # north-star tolerance (we expect and assert bit-exact below)


def assert_same(tag, g_ids, g_dist, g_cnt, g_sc, r_ids, r_dist, r_cnt, r_sc):
    g_ids, g_dist = np.asarray(g_ids), np.asarray(g_dist)
    np.testing.assert_array_equal(np.asarray(g_cnt), r_cnt, err_msg=f"{tag}: count")
    if r_sc is not None and g_sc is not None:
        np.testing.assert_array_equal(np.asarray(g_sc), r_sc, err_msg=f"{tag}: scanned_vectors")
    for q in range(len(r_cnt)):
        c = int(r_cnt[q])
        np.testing.assert_array_equal(g_ids[q, :c], r_ids[q, :c], err_msg=f"{tag}: ids q={q}")
        a, b = g_dist[q, :c], r_dist[q, :c]
        rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-30)
        assert (rel <= MAXREL).all(), f"{tag}: dist rel err {rel.max()} q={q}"
        np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32), err_msg=f"{tag}: dist bits q={q}")


@pytest.fixture(scope="module")
def gpu():
    if pg.device_count() < 1:
        pytest.skip("no CUDA device")
    return 0


@pytest.mark.parametrize("path_mode", [0, 1], ids=["auto", "generic"])
@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_golden_reference_parity(gpu, case, path_mode):
    path, z, grid = load_golden(case)
    ix = pg.GpuIndex.load(path, gpu)
    ix.set_scan_path(path_mode)
    q = z["queries"]
    for nprobe, k in grid:
        key = f"p{nprobe}_k{k}"
        r = ix.search_batch(q, k, nprobe)
        assert_same(f"{case}/{key}", r.ids, r.dist, r.count, r.scanned, z[key + "_ids"], z[key + "_dist"],
                    z[key + "_count"], z[key + "_scanned"])


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_probe_lists_match_oracle(gpu, case):
    path, z, grid = load_golden(case)
    ix = pg.GpuIndex.load(path, gpu)
    oi = O.OracleIndex(path)
    q = z["queries"]
    for nprobe in sorted({g[0] for g in grid} | {ix.nlist}):
        lists, dist = ix.probe(q, nprobe)
        for i in range(q.shape[0]):
            ol, od = oi.probe_lists(q[i], nprobe)
            np.testing.assert_array_equal(lists[i], ol)
            np.testing.assert_array_equal(dist[i].view(np.uint32), od.view(np.uint32))


def test_validation_errors_match_reference(gpu):
    """test_annindex.cpp:176-192 (search part)."""
    path, z, _ = load_golden("rand600_d16")
    ix = pg.GpuIndex.load(path, gpu)
    q = z["queries"][:1]
    with pytest.raises(pg.ConfigError, match="nprobe out of"):
        ix.search_batch(q, 1, 0)
    with pytest.raises(pg.ConfigError, match="nprobe out of"):
        ix.search_batch(q, 1, ix.nlist + 1)
    with pytest.raises(pg.ConfigError, match="k must be"):
        ix.search_batch(q, 0, 1)
    with pytest.raises(pg.ConfigError):
        pg.search(ix, q[0], pg.SearchParams(1, 1, True))


def test_load_errors(gpu, tmp_path):
    with pytest.raises(pg.FormatError, match="cannot open"):
        pg.GpuIndex.load(str(tmp_path / "missing.bin"), gpu)
    p = tmp_path / "bad.bin"
    src = open(load_golden("rand600_d16")[0], "rb").read()
    p.write_bytes(b"XXXX" + src[4:])
    with pytest.raises(pg.FormatError, match="bad index magic at offset 0"):
        pg.GpuIndex.load(str(p), gpu)
    for cut in (3, 10, 5000):
        p.write_bytes(src[:-cut])
        with pytest.raises(pg.FormatError) as e:
            pg.GpuIndex.load(str(p), gpu)
        with pytest.raises(O.OracleError) as eo:
            O.OracleIndex(str(p))
        assert str(e.value) == str(eo.value)


def test_single_query_api_and_kats(gpu):
    """test_annindex.cpp:60-71 (four points) and :127-143 (scanned counts)."""
    path, z, _ = load_golden("four_points")
    ix = pg.GpuIndex.load(path, gpu)
    for i in range(4):
        r = pg.search(ix, z["queries"][i], pg.SearchParams(nprobe=4, k=1))
        assert len(r.neighbors) == 1 and r.neighbors[0].chunk_id == i and r.scanned_lists == 4
    path, z, _ = load_golden("two_clusters")
    ix = pg.GpuIndex.load(path, gpu)
    q = np.zeros(8, np.float32)
    q[0] = -10
    r = pg.search(ix, q, pg.SearchParams(nprobe=1, k=5))
    assert r.scanned_lists == 1 and r.scanned_vectors == 100
    assert all(n.chunk_id < 100 for n in r.neighbors)
    assert pg.search(ix, q, pg.SearchParams(nprobe=2, k=5)).scanned_vectors == 200


@pytest.fixture(scope="module")
def synth(gpu, tmp_path_factory):
    from paper_2403_05676_b200 import fixtures as F
    os.environ.setdefault("PRAG_FIXTURE_DIR", str(tmp_path_factory.mktemp("fx")))
    out = {}
    for nsq in (32, 64):
        p, q, meta = F.ensure_fixture(300_000, 384, 256, nsq, seed=5 + nsq, nq=64, log=lambda *a: None)
        out[nsq] = (p, q)
    return out


@pytest.mark.parametrize("path_mode", [0, 1], ids=["auto", "generic"])
@pytest.mark.parametrize("nsq", [32, 64])
def test_synthetic_oracle_parity(synth, nsq, path_mode):
    p, q = synth[nsq]
    ix = pg.GpuIndex.load(p, 0)
    ix.set_scan_path(path_mode)
    assert ix.desc.code_layout == 1
    oi = O.OracleIndex(p)
    for nprobe, k in [(1, 10), (16, 10), (16, 1), (64, 100), (7, 2), (256, 10), (16, 32), (16, 33), (3, 31)]:
        r = ix.search_batch(q, k, nprobe)
        o = oi.search(q, nprobe, k)
        assert_same(f"synth{nsq}/p{nprobe}k{k}", r.ids, r.dist, r.count, r.scanned, *o)


def test_device_pointers_and_streams(synth):
    import torch
    p, q = synth[32]
    ix = pg.GpuIndex.load(p, 0)
    host = ix.search_batch(q, 10, 16)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        dq = torch.from_numpy(q).cuda()
        dev = ix.search_batch(dq, 10, 16)
    s.synchronize()
    assert_same("device", dev.ids.cpu().numpy().view(np.uint64), dev.dist.cpu().numpy(),
                dev.count.cpu().numpy().view(np.uint32), dev.scanned.cpu().numpy().view(np.uint64),
                host.ids, host.dist, host.count, host.scanned)


def test_repeated_search_bit_identical(synth):
    """acceptance.cpp C9 (:397-440): repeated search is bit-identical."""
    p, q = synth[64]
    ix = pg.GpuIndex.load(p, 0)
    a = ix.search_batch(q, 10, 32)
    for _ in range(3):
        b = ix.search_batch(q, 10, 32)
        assert_same("repeat", b.ids, b.dist, b.count, b.scanned, a.ids, a.dist, a.count, a.scanned)


def test_concurrent_searches(synth):
    """One index shared by threads on distinct streams (service.hpp:303-354)."""
    import torch
    p, q = synth[32]
    ix = pg.GpuIndex.load(p, 0)
    ref = ix.search_batch(q, 10, 8)
    errs = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            for _ in range(5):
                with torch.cuda.stream(s):
                    r = ix.search_batch(q, 10, 8)
                assert_same(f"thread{i}", r.ids, r.dist, r.count, r.scanned, ref.ids, ref.dist, ref.count,
                            ref.scanned)
        except Exception as e:
            errs.append(e)
    th = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errs, errs[0]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_search_merge_equals_unsharded(synth, world):
    """list-sharded search + exact merge == unsharded search."""
    import torch
    p, q = synth[32]
    full = pg.GpuIndex.load(p, 0)
    k, nprobe = 10, 16
    ref = full.search_batch(q, k, nprobe)
    shards = [pg.GpuIndex.load_shard(p, r, world, 0) for r in range(world)]
    assert sum(s.ntotal for s in shards) == full.ntotal
    parts = [s.search_batch(torch.from_numpy(q).cuda(), k, nprobe) for s in shards]
    ids = torch.stack([x.ids for x in parts])
    dist = torch.stack([x.dist for x in parts])
    cnt = torch.stack([x.count for x in parts])
    sc = torch.stack([x.scanned for x in parts])
    m = pg.merge_topk(ids, dist, cnt, sc, k)
    torch.cuda.synchronize()
    assert_same(f"shard{world}", m.ids.cpu().numpy().view(np.uint64), m.dist.cpu().numpy(),
                m.count.cpu().numpy().view(np.uint32), m.scanned.cpu().numpy().view(np.uint64),
                ref.ids, ref.dist, ref.count, ref.scanned)


def test_batch_edges(synth):
    p, q = synth[32]
    ix = pg.GpuIndex.load(p, 0)
    r = ix.search_batch(q[:0], 10, 4)
    assert r.ids.shape == (0, 10)
    oi = O.OracleIndex(p)
    # k far above the candidate count: fewer results, no padding
    r = ix.search_batch(q[:3], 5000, 1)
    o = oi.search(q[:3], 1, 5000)
    assert_same("bigk", r.ids, r.dist, r.count, r.scanned, *o)


# ----------------------------------------------------- tensor-core coarse K1
def _probe_both(ix, q, nprobe):
    ix.set_coarse_path(0)
    a = ix.probe(q, nprobe)
    ix.set_coarse_path(1)
    b = ix.probe(q, nprobe)
    ix.set_coarse_path(0)
    return a, b


@pytest.mark.parametrize("threads", ["512", "1024"])
@pytest.mark.parametrize("nsq", [32, 64])
def test_tc_coarse_probe_lists_exact(synth, nsq, threads, monkeypatch):
    """K1 tcgen05 pre-filter + exact window rescoring == exact SIMT coarse ==
    the oracle's sequential squared_l2 order (annindex.hpp:277-281), with
    K1b at both block sizes."""
    monkeypatch.setenv("PRAG_GPU_K1B_THREADS", threads)
    p, q = synth[nsq]
    ix = pg.GpuIndex.load(p, 0)
    oi = O.OracleIndex(p)
    # 120-129: K1b windows on both sides of the one-batch rescoring limit
    # (2 x 64 staged rows at d = 384)
    for nprobe in (1, 2, 16, 64, 120, 124, 126, 127, 128, 129, 200, 256):
        (tl, td), (el, ed) = _probe_both(ix, q, nprobe)
        assert (tl == el).all(), f"nprobe={nprobe}: TC probe lists differ from exact"
        assert (td.view(np.uint32) == ed.view(np.uint32)).all()
        for i in range(0, q.shape[0], 7):
            ol, od = oi.probe_lists(q[i], nprobe)
            assert (tl[i] == ol).all() and (td[i].view(np.uint32) == od.view(np.uint32)).all()


def _adversarial_index(tmp_path, nlist=256, d=64, nsq=16, dup=8, seed=3):
    """Duplicated centroids (exact distance ties across lists), a far-away
    cluster of centroids (large norms), and queries sitting exactly on
    centroids (distance 0: A - E < 0)."""
    rng = np.random.default_rng(seed)
    cent = rng.standard_normal((nlist, d)).astype(np.float32)
    for i in range(0, nlist, dup):  # blocks of identical centroids
        cent[i:i + dup // 2] = cent[i]
    cent[-32:] += np.float32(40.0)
    words = rng.standard_normal((nsq, 256, d // nsq)).astype(np.float32) * np.float32(0.1)
    lists = []
    nid = 0
    for l in range(nlist):
        n = int(rng.integers(0, 40))
        lists.append((np.arange(nid, nid + n, dtype=np.uint64), rng.integers(0, 256, (n, nsq), dtype=np.uint8)))
        nid += n
    p = str(tmp_path / "adv.pragix")
    O.write_pragix(p, cent, words, lists)
    q = np.concatenate([cent[:40], cent[:20] + np.float32(1e-3), rng.standard_normal((40, d)).astype(np.float32),
                        cent[-8:] * np.float32(1.0001)]).astype(np.float32)
    return p, q


@pytest.mark.parametrize("nlist,threads", [(256, None), (256, "1024"), (4096, "512"), (4096, "1024"),
                                           (16384, "512"), (16384, "1024")])
def test_tc_coarse_adversarial_ties(gpu, tmp_path, nlist, threads, monkeypatch):
    """Also at the benchmarked list counts, where K1b holds 4-32 keys per
    thread (every select_window_kernel<VPT, threads> instantiation in use)."""
    if threads:
        monkeypatch.setenv("PRAG_GPU_K1B_THREADS", threads)
    p, q = _adversarial_index(tmp_path, nlist=nlist)
    ix = pg.GpuIndex.load(p, gpu)
    oi = O.OracleIndex(p)
    for nprobe in (1, 3, 4, 5, 17, 128, 256):
        (tl, td), (el, ed) = _probe_both(ix, q, nprobe)
        assert (tl == el).all() and (td.view(np.uint32) == ed.view(np.uint32)).all(), f"nprobe={nprobe}"
        for i in range(q.shape[0]):
            ol, _ = oi.probe_lists(q[i], nprobe)
            assert (tl[i] == ol).all(), (nprobe, i)
    # full search through the TC path against the oracle
    for nprobe, k in [(4, 10), (64, 5)]:
        r = ix.search_batch(q, k, nprobe)
        assert_same(f"adv/p{nprobe}", r.ids, r.dist, r.count, r.scanned, *oi.search(q, nprobe, k))


def test_tc_coarse_large_batch(synth):
    """nq > 256 spans several N tiles of the tcgen05 GEMM."""
    p, q = synth[32]
    ix = pg.GpuIndex.load(p, 0)
    rng = np.random.default_rng(1)
    qq = (q[rng.integers(0, q.shape[0], 600)] + rng.standard_normal((600, q.shape[1])).astype(np.float32) *
          np.float32(0.3)).astype(np.float32)
    (tl, td), (el, ed) = _probe_both(ix, qq, 16)
    assert (tl == el).all() and (td.view(np.uint32) == ed.view(np.uint32)).all()
