"""The batch-1 single-launch search (csrc/batch1.cu: coarse, probe selection,
ADC tables, scan and merge in one cooperative grid with two grid barriers)
against the reference semantics (annindex.hpp:262-315): the golden fixtures
written by the unmodified reference, the CPU oracle on seeded fixtures, the
exact restatement of the device-built synthetic index, and the five-kernel
chain. The kernel is opt-in (PRAG_GPU_BATCH1=1, set for this module; the
chain is measured faster, batch1.cu). Bit-exact on
ids, distance bits, count and scanned_vectors, including exact distance ties,
empty lists, k above the candidate count and captured plans."""
import os

import numpy as np
import pytest

import _oracle as O
import _synth_ref as R
from conftest import GOLDEN_CASES, load_golden
from test_gpu_parity import assert_same

pg = pytest.importorskip("paper_2403_05676_b200")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def batch1_on():
    os.environ["PRAG_GPU_BATCH1"] = "1"
    yield
    os.environ.pop("PRAG_GPU_BATCH1", None)


@pytest.fixture(scope="module")
def gpu():
    if pg.device_count() < 1:
        pytest.skip("no CUDA device")
    return 0


def chain(ix, q, k, nprobe):
    os.environ["PRAG_GPU_BATCH1"] = "0"
    try:
        return ix.search_batch(q, k, nprobe)
    finally:
        os.environ["PRAG_GPU_BATCH1"] = "1"


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_golden_batch1(gpu, case):
    path, z, grid = load_golden(case)
    ix = pg.GpuIndex.load(path, 0)
    if ix.desc.code_layout != 1:
        pytest.skip("generic code layout (m not in {32, 64}): batch-1 kernel not used")
    q = z["queries"]
    oi = O.OracleIndex(path)
    for nprobe, k in grid:
        for i in range(q.shape[0]):
            r = ix.search_batch(q[i:i + 1], k, nprobe)
            assert_same(f"{case}/p{nprobe}k{k}/q{i}", r.ids, r.dist, r.count, r.scanned, *oi.search(q[i:i + 1], nprobe, k))
            key = f"p{nprobe}_k{k}"
            c = int(r.count[0])
            assert (r.ids[0, :c] == z[key + "_ids"][i, :c]).all()


@pytest.fixture(scope="module")
def fx(gpu, tmp_path_factory):
    from paper_2403_05676_b200 import fixtures as F
    os.environ.setdefault("PRAG_FIXTURE_DIR", str(tmp_path_factory.mktemp("fx1")))
    out = {}
    for nsq, nlist in ((32, 256), (64, 1024)):
        p, q, _ = F.ensure_fixture(300_000, 384, nlist, nsq, seed=11 + nsq, nq=32, log=lambda *a: None)
        out[nsq] = (p, q)
    return out


@pytest.mark.parametrize("nsq", [32, 64])
def test_oracle_and_chain_batch1(fx, nsq):
    path, q = fx[nsq]
    ix = pg.GpuIndex.load(path, 0)
    oi = O.OracleIndex(path)
    for nprobe, k in ((1, 1), (1, 10), (7, 2), (16, 32), (64, 10), (64, 32)):
        for i in range(0, q.shape[0], 3):
            r = ix.search_batch(q[i:i + 1], k, nprobe)
            tag = f"m{nsq}/p{nprobe}k{k}/q{i}"
            assert_same(tag, r.ids, r.dist, r.count, r.scanned, *oi.search(q[i:i + 1], nprobe, k))
            c = chain(ix, q[i:i + 1], k, nprobe)
            assert_same(tag + "/chain", r.ids, r.dist, r.count, r.scanned, c.ids, c.dist, c.count, c.scanned)


def test_batch1_device_plan_and_repeat(fx):
    import torch
    path, q = fx[32]
    ix = pg.GpuIndex.load(path, 0)
    oi = O.OracleIndex(path)
    dq = torch.from_numpy(q[5:6].copy()).cuda()
    out = pg.BatchResult(torch.empty((1, 2), dtype=torch.int64, device="cuda"),
                         torch.empty((1, 2), dtype=torch.float32, device="cuda"),
                         torch.empty((1,), dtype=torch.int32, device="cuda"),
                         torch.empty((1,), dtype=torch.int64, device="cuda"))
    plan = ix.plan(dq, 2, 16, out)
    want = oi.search(q[5:6], 16, 2)
    for rep in range(20):  # graph replays: barrier and ticket counters return to their start state
        plan.launch()
        torch.cuda.synchronize()
        assert_same(f"plan/{rep}", out.ids.cpu().numpy().view(np.uint64), out.dist.cpu().numpy(),
                    out.count.cpu().numpy().view(np.uint32), out.scanned.cpu().numpy().view(np.uint64), *want)
    for i in range(q.shape[0]):  # new queries through the same buffer
        dq.copy_(torch.from_numpy(q[i:i + 1]))
        plan.launch()
        torch.cuda.synchronize()
        assert_same(f"plan/q{i}", out.ids.cpu().numpy().view(np.uint64), out.dist.cpu().numpy(),
                    out.count.cpu().numpy().view(np.uint32), out.scanned.cpu().numpy().view(np.uint64),
                    *oi.search(q[i:i + 1], 16, 2))


@pytest.mark.parametrize("m", [32, 64])
def test_synthetic_batch1(gpu, m):
    rng = np.random.default_rng(9)
    nlist, d = 2048, 384
    cents = rng.standard_normal((nlist, d)).astype(np.float32)
    words = (rng.standard_normal((m, 256, d // m)) * 0.3).astype(np.float32)
    seed = 400 + m
    ix = pg.GpuIndex.synthetic(cents, words, 2_000_000, seed=seed, sigma=1.0)
    sizes = ix.list_sizes()
    q = (cents[rng.integers(0, nlist, 4)] + rng.standard_normal((4, d)).astype(np.float32) * 0.5).astype(np.float32)
    for nprobe, k in ((1, 2), (16, 2), (64, 32)):
        for i in range(q.shape[0]):
            r = ix.search_batch(q[i:i + 1], k, nprobe)
            ids, dist, sc = R.search(q[i], cents, words, sizes, seed, nprobe, k)
            c = int(r.count[0])
            assert c == len(ids) and int(r.scanned[0]) == sc
            assert (r.ids[0, :c] == ids).all()
            assert (r.dist[0, :c].view(np.uint32) == dist.view(np.uint32)).all()


def test_batch1_ties_between_ctas(gpu, tmp_path):
    """Many exact distance ties spread over the lists (identical codes), so
    the final merge of the per-CTA lists has to order by chunk id."""
    rng = np.random.default_rng(3)
    nlist, d, m = 64, 64, 32
    cents = rng.standard_normal((nlist, d)).astype(np.float32)
    words = rng.standard_normal((m, 256, d // m)).astype(np.float32)
    n = 40_000
    assign = rng.integers(0, nlist, n)
    order = np.argsort(assign, kind="stable")
    list_off = np.zeros(nlist + 1, np.uint64)
    np.add.at(list_off, assign + 1, 1)
    list_off = np.cumsum(list_off).astype(np.uint64)
    ids = rng.permutation(n).astype(np.uint64)[order]
    codes = np.repeat(rng.integers(0, 256, (1, m)).astype(np.uint8), n, axis=0)  # every entry the same code
    codes[::7] = rng.integers(0, 256, (len(codes[::7]), m))
    from paper_2403_05676_b200 import fixtures as F
    p = str(tmp_path / "ties.pragix")
    F.write_pragix(p, cents, words, list_off, ids, codes)
    ix = pg.GpuIndex.load(p, 0)
    oi = O.OracleIndex(p)
    q = cents[:3] + 0.01
    for nprobe, k in ((8, 32), (64, 32), (3, 5)):
        for i in range(q.shape[0]):
            r = ix.search_batch(q[i:i + 1], k, nprobe)
            assert_same(f"ties/p{nprobe}k{k}/q{i}", r.ids, r.dist, r.count, r.scanned, *oi.search(q[i:i + 1], nprobe, k))
