"""GPU parity at the shapes that are benchmarked (SURVEY.md 8a rows a4-a7,
annindex.hpp:277-313), against the CPU oracle, bit-exact on ids, distances,
counts and scanned_vectors:

  * config B itself -- 10M x 384, nlist 4096, m 32: the bench's own fixture
    and 64 queries, nprobe {1, 16, 128} x k {2, 10, 32}. Its largest list
    (21k entries) is split into several scan work items;
  * an nlist sweep {1024 .. 16384} at 2M entries, so every instantiation of
    the tensor-core window select (select_window_kernel<2/4/8/16/32>,
    coarse_tc.cu) runs, with the probe lists checked too;
  * a config-C slice: m 64, nlist 16384 (the config C/D layout) at 4M.

Fixtures are GPU-built PRAGIX01 files (paper_2403_05676_b200/fixtures.py)
that the oracle reads byte for byte."""
import os

import numpy as np
import pytest

import _oracle as O
from test_gpu_parity import assert_same

pg = pytest.importorskip("paper_2403_05676_b200")
pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


def _fixture(n, nlist, nsq, seed, nq=64):
    from paper_2403_05676_b200 import fixtures as F
    if pg.device_count() < 1:
        pytest.skip("no CUDA device")
    return F.ensure_fixture(n, 384, nlist, nsq, seed=seed, nq=nq, log=lambda *a: None)


@pytest.fixture(scope="module")
def config_b():
    # the same fixture bench.py times (CFG: n 10M, nlist 4096, m 32, seed 1, 64 queries)
    p, q, meta = _fixture(10_000_000, 4096, 32, 1)
    ix = pg.GpuIndex.load(p, 0)
    oi = O.OracleIndex(p)
    return ix, oi, q, meta


@pytest.mark.parametrize("nprobe", [1, 16, 128])
def test_config_b_parity(config_b, nprobe):
    ix, oi, q, meta = config_b
    assert meta["list_max"] > 16384  # the largest list spans several scan items
    for k in (2, 10, 32):
        r = ix.search_batch(q, k, nprobe)
        o = oi.search(q, nprobe, k, threads=THREADS)
        assert_same(f"B/p{nprobe}k{k}", r.ids, r.dist, r.count, r.scanned, *o)


def test_config_b_batch1_and_device_plan(config_b):
    """The pipeline's call shape (one query, k = 2: pipeline.hpp:228) and the
    captured plan the bench times, against the oracle."""
    import torch
    ix, oi, q, _ = config_b
    for i in (0, 17, 63):
        r = ix.search_batch(q[i:i + 1], 2, 16)
        assert_same(f"B/q{i}", r.ids, r.dist, r.count, r.scanned, *oi.search(q[i:i + 1], 16, 2))
    dq = torch.from_numpy(q).cuda()
    out = pg.BatchResult(torch.empty((64, 10), dtype=torch.int64, device="cuda"),
                         torch.empty((64, 10), dtype=torch.float32, device="cuda"),
                         torch.empty((64,), dtype=torch.int32, device="cuda"),
                         torch.empty((64,), dtype=torch.int64, device="cuda"))
    plan = ix.plan(dq, 10, 16, out)
    for _ in range(3):
        plan.launch()
    torch.cuda.synchronize()
    assert_same("B/plan", out.ids.cpu().numpy().view(np.uint64), out.dist.cpu().numpy(),
                out.count.cpu().numpy().view(np.uint32), out.scanned.cpu().numpy().view(np.uint64),
                *oi.search(q, 16, 10, threads=THREADS))


@pytest.mark.parametrize("nlist", [1024, 2048, 4096, 8192, 16384])
def test_nlist_sweep_parity(nlist):
    p, q, _ = _fixture(2_000_000, nlist, 32, 40 + nlist % 97)
    ix = pg.GpuIndex.load(p, 0)
    oi = O.OracleIndex(p)
    for nprobe in (1, 16, 256):
        lists, dist = ix.probe(q, nprobe)
        for i in range(0, q.shape[0], 9):
            ol, od = oi.probe_lists(q[i], nprobe)
            np.testing.assert_array_equal(lists[i], ol, err_msg=f"nlist={nlist} nprobe={nprobe} q={i}")
            np.testing.assert_array_equal(dist[i].view(np.uint32), od.view(np.uint32))
    for nprobe, k in ((16, 10), (200, 10), (64, 32)):
        r = ix.search_batch(q, k, nprobe)
        assert_same(f"L{nlist}/p{nprobe}k{k}", r.ids, r.dist, r.count, r.scanned,
                    *oi.search(q, nprobe, k, threads=THREADS))


def test_config_c_slice_m64_nlist16384():
    p, q, meta = _fixture(4_000_000, 16384, 64, 77)
    ix = pg.GpuIndex.load(p, 0)
    assert ix.desc.code_layout == 1
    oi = O.OracleIndex(p)
    for nprobe, k in ((1, 10), (16, 10), (128, 10), (64, 32), (16, 2)):
        r = ix.search_batch(q, k, nprobe)
        assert_same(f"C/p{nprobe}k{k}", r.ids, r.dist, r.count, r.scanned,
                    *oi.search(q, nprobe, k, threads=THREADS))
    for i in (0, 31):  # batch 1
        r = ix.search_batch(q[i:i + 1], 10, 64)
        assert_same(f"C/q{i}", r.ids, r.dist, r.count, r.scanned, *oi.search(q[i:i + 1], 64, 10))
