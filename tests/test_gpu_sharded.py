"""List-sharded search through the C ABI, on one GPU.

Every gpurun box has one B200, so shards share device 0 here; the code path is
the multi-device one (per-shard streams, per-shard passes, the root merge
kernel reading each shard's top-k block in place, cross-stream events) --
only the peer copies for GPUs without peer access are not exercised.

  * group handles (one process): prag_gpu_index_load_sharded / _group /
    _synthetic_shard over 2..8 shards == the unsharded index == the oracle,
    through prag_gpu_search (host and device pointers), plans, rerank;
  * a distributed shard (prag_gpu_comm, NCCL) at world 1: the collective
    search (local pass + ncclAllGather + merge) and its captured plan, and
    the torch.distributed rendezvous of the unique id (ShardedIndex).

The bar is the unsharded search's bits: ids, distances, counts and
scanned_vectors identical."""
import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import _oracle as O  # noqa: E402
from test_gpu_parity import assert_same  # noqa: E402

pg = pytest.importorskip("paper_2403_05676_b200")
pytestmark = pytest.mark.gpu


def _res(r):
    import torch
    if isinstance(r.ids, torch.Tensor):
        return (r.ids.cpu().numpy().view(np.uint64), r.dist.cpu().numpy(), r.count.cpu().numpy().view(np.uint32),
                r.scanned.cpu().numpy().view(np.uint64))
    return r.ids, r.dist, r.count, r.scanned


def _same(tag, a, b):
    assert_same(tag, *_res(a), *_res(b))


@pytest.fixture(scope="module")
def fx():
    from paper_2403_05676_b200 import fixtures as F
    if pg.device_count() < 1:
        pytest.skip("no CUDA device")
    p, q, _ = F.ensure_fixture(300_000, 384, 256, 32, seed=37, nq=64, log=lambda *a: None)
    return p, q, pg.GpuIndex.load(p, 0)


GRID = [(16, 10), (1, 10), (64, 32), (256, 2), (16, 100)]  # k = 100: the generic scan path


@pytest.mark.parametrize("world", [2, 3, 8])
def test_load_sharded_group_equals_unsharded(fx, world):
    p, q, full = fx
    g = pg.GpuIndex.load_sharded(p, [0] * world)
    assert g.desc.shard_world == world and g.ntotal == full.ntotal
    assert (g.list_sizes() == full.list_sizes()).all()
    for nprobe, k in GRID:
        _same(f"group{world}/p{nprobe}k{k}", g.search_batch(q, k, nprobe), full.search_batch(q, k, nprobe))
    oi = O.OracleIndex(p)
    r = g.search_batch(q, 10, 16)
    assert_same(f"group{world}/oracle", r.ids, r.dist, r.count, r.scanned, *oi.search(q, 16, 10))
    a, b = g.probe(q, 16), full.probe(q, 16)
    assert (a[0] == b[0]).all()


def test_group_device_pointers_plan_and_streams(fx):
    import torch
    p, q, full = fx
    g = pg.GpuIndex.load_sharded(p, [0, 0, 0, 0])
    ref = full.search_batch(q, 10, 16)
    s = torch.cuda.Stream()
    dq = torch.from_numpy(q).cuda()
    with torch.cuda.stream(s):
        dev = g.search_batch(dq, 10, 16)
    s.synchronize()
    _same("group/device", dev, ref)
    out = pg.BatchResult(torch.empty((64, 10), dtype=torch.int64, device="cuda"),
                         torch.empty((64, 10), dtype=torch.float32, device="cuda"),
                         torch.empty((64,), dtype=torch.int32, device="cuda"),
                         torch.empty((64,), dtype=torch.int64, device="cuda"))
    plan = g.plan(dq, 10, 16, out, stream=s)
    for i in range(3):  # replays; new queries written into the plan's buffer in between
        plan.launch(stream=s)
        s.synchronize()
        _same(f"group/plan{i}", out, ref)
    dq.copy_(torch.from_numpy(q[::-1].copy()))
    plan.launch(stream=s)
    s.synchronize()
    _same("group/plan-new-queries", out, full.search_batch(q[::-1].copy(), 10, 16))


def test_group_concurrent_callers(fx):
    """Threads share one group handle (service.hpp:303-354)."""
    import threading
    p, q, full = fx
    g = pg.GpuIndex.load_sharded(p, [0, 0, 0])
    ref = full.search_batch(q, 10, 8)
    errs = []

    def worker(i):
        import torch
        try:
            s = torch.cuda.Stream()
            for _ in range(4):
                with torch.cuda.stream(s):
                    _same(f"thread{i}", g.search_batch(q, 10, 8), ref)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errs, errs[0]


def test_group_of_shard_handles(fx):
    p, q, full = fx
    shards = [pg.GpuIndex.load_shard(p, r, 3, 0) for r in (2, 0, 1)]  # any order: placed by rank
    g = pg.GpuIndex.group(shards)
    assert all(s._h is None for s in shards)
    _same("group-of-shards", g.search_batch(q, 10, 32), full.search_batch(q, 10, 32))
    with pytest.raises(pg.ConfigError):  # ranks must be 0..n-1 of one world
        pg.GpuIndex.group([pg.GpuIndex.load_shard(p, 0, 2, 0)])


def test_group_rerank_and_calibration():
    """exact_rerank (annindex.hpp:307-312) on a group: every shard reranks its
    candidates, the merge keeps the full-precision order."""
    sys.path.insert(0, os.path.join(HERE, "golden"))
    import make_train_golden as M
    name = "d64_m16"
    path = os.path.join(HERE, "golden", name + ".pragix")
    v = M.vectors({c["name"]: c["gen"] for c in M.EXISTING}[name])
    q = np.load(os.path.join(HERE, "golden", name + ".npz"))["queries"]
    full = pg.GpuIndex.load(path, 0)
    full.set_embeddings(v)
    g = pg.GpuIndex.load_sharded(path, [0, 0])
    g.set_embeddings(v)
    for nprobe, k in ((4, 10), (full.nlist, 50)):
        _same(f"rerank/p{nprobe}", g.search_batch(q, k, nprobe, exact_rerank=True),
              full.search_batch(q, k, nprobe, exact_rerank=True))
    m, lat = pg.calibrate_gpu(g, q[:4], 2, [1, 4, 16], repeats=3, warmups=1)
    assert len(lat) == 3 and m.slope_s >= 0


def _model(nlist, d, m, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((nlist, d)).astype(np.float32),
            (rng.standard_normal((m, 256, d // m)) * 0.3).astype(np.float32))


@pytest.mark.parametrize("m", [32, 64])
def test_synthetic_shards_equal_full_synthetic(m):
    cents, words = _model(512, 384, m, 9)
    n, seed = 400_000, 5 + m
    full = pg.GpuIndex.synthetic(cents, words, n, seed=seed, sigma=1.0)
    world = 4
    shards = [pg.GpuIndex.synthetic_shard(cents, words, n, r, world, seed=seed, sigma=1.0) for r in range(world)]
    assert sum(s.ntotal for s in shards) == n
    assert (sum(s.list_sizes() for s in shards) == full.list_sizes()).all()
    g = pg.GpuIndex.group(shards)
    rng = np.random.default_rng(3)
    q = (cents[rng.integers(0, 512, 32)] + rng.standard_normal((32, 384)).astype(np.float32) * 0.5).astype(np.float32)
    for nprobe, k in ((1, 10), (16, 10), (64, 32)):
        _same(f"synth{m}/p{nprobe}k{k}", g.search_batch(q, k, nprobe), full.search_batch(q, k, nprobe))


def test_nccl_comm_world1_collective_search_and_plan():
    """A distributed shard at world 1: prag_gpu_search on it is the collective
    path (local pass, ncclAllGather of the top-k block, merge kernel), and its
    plan captures the NCCL call in the graph."""
    import torch
    cents, words = _model(256, 384, 64, 4)
    n, seed = 200_000, 17
    full = pg.GpuIndex.synthetic(cents, words, n, seed=seed)
    shard = pg.GpuIndex.synthetic_shard(cents, words, n, 0, 1, seed=seed)
    comm = pg.Comm(pg.Comm.unique_id(), 1, 0, 0)
    shard.attach_comm(comm)
    rng = np.random.default_rng(5)
    q = (cents[rng.integers(0, 256, 16)] + rng.standard_normal((16, 384)).astype(np.float32) * 0.5).astype(np.float32)
    _same("nccl/host", shard.search_batch(q, 10, 16), full.search_batch(q, 10, 16))
    dq = torch.from_numpy(q).cuda()
    out = pg.BatchResult(torch.empty((16, 10), dtype=torch.int64, device="cuda"),
                         torch.empty((16, 10), dtype=torch.float32, device="cuda"),
                         torch.empty((16,), dtype=torch.int32, device="cuda"),
                         torch.empty((16,), dtype=torch.int64, device="cuda"))
    plan = shard.plan(dq, 10, 16, out)
    plan.launch()
    torch.cuda.synchronize()
    _same("nccl/plan", out, full.search_batch(q, 10, 16))
    with pytest.raises(pg.ConfigError):  # comm rank/world must match the shard
        pg.GpuIndex.synthetic_shard(cents, words, n, 1, 2, seed=seed).attach_comm(comm)
    plan.close()
    shard.attach_comm(None)
    comm.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_sharded_index_over_torch_distributed(fx):
    """ShardedIndex: the unique id travels over torch.distributed, the
    exchange itself is libprag_gpu's ncclAllGather."""
    import torch.distributed as dist

    from paper_2403_05676_b200 import distributed as D
    p, q, full = fx
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        si = D.ShardedIndex.load(p, device=0)
        _same("ShardedIndex", si.search_batch(q, 10, 16), full.search_batch(q, 10, 16))
        si.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["d384_m32", "d384_m64"])
def test_striped_lists_equal_unsharded(tmp_path, name):
    """Large lists striped over the shards (plan_shard_ranges): list 0 holds 4
    copies of every entry (new ids, same codes), so it is striped at every
    world here and its stripes hold exact distance ties with each other. The
    group (load_sharded), shard handles (load_shard, read by entry range) and
    the oracle on the unsharded file agree bit for bit."""
    from test_multiproc_cpu import _skewed_pragix
    src = os.path.join(HERE, "golden", name + ".pragix")
    path = str(tmp_path / "skew.pragix")
    sizes = _skewed_pragix(src, path)
    q = np.load(os.path.join(HERE, "golden", name + ".npz"))["queries"]
    full = pg.GpuIndex.load(path, 0)
    oi = O.OracleIndex(path)
    for world in (2, 3, 8):
        assert pg.plan_shards(sizes, world)[0] == world
        g = pg.GpuIndex.load_sharded(path, [0] * world)
        assert (g.list_sizes() == full.list_sizes()).all()
        h = pg.GpuIndex.group([pg.GpuIndex.load_shard(path, r, world, 0) for r in range(world)])
        for nprobe, k in ((32, 10), (4, 32), (1, 10), (32, 100)):
            ref = full.search_batch(q, k, nprobe)
            _same(f"{name}/stripe{world}/p{nprobe}k{k}", g.search_batch(q, k, nprobe), ref)
            _same(f"{name}/stripe{world}/shards/p{nprobe}k{k}", h.search_batch(q, k, nprobe), ref)
        r = g.search_batch(q, 10, 32)
        assert_same(f"{name}/stripe{world}/oracle", r.ids, r.dist, r.count, r.scanned, *oi.search(q, 32, 10))


def test_synthetic_striped_shards_equal_full_synthetic():
    """Synthetic shards with a heavy list-size skew: the largest lists are
    striped (each stripe keeps its entries' global chunk ids and codes)."""
    cents, words = _model(256, 384, 64, 11)
    n, seed, sigma = 600_000, 21, 1.6
    full = pg.GpuIndex.synthetic(cents, words, n, seed=seed, sigma=sigma)
    sizes = full.list_sizes()
    for world in (2, 4):
        owner = pg.plan_shards(sizes, world)
        assert (owner == world).sum() >= 3
        shards = [pg.GpuIndex.synthetic_shard(cents, words, n, r, world, seed=seed, sigma=sigma) for r in range(world)]
        for r, s in enumerate(shards):
            b, e = pg.plan_shard_ranges(sizes, world, r)
            assert (s.list_sizes() == e - b).all()
        g = pg.GpuIndex.group(shards)
        big = np.argsort(-sizes.astype(np.int64))[:8]  # queries at the largest lists' centroids
        rng = np.random.default_rng(4)
        q = (cents[np.concatenate([big, rng.integers(0, 256, 8)])] +
             rng.standard_normal((16, 384)).astype(np.float32) * 0.3).astype(np.float32)
        for nprobe, k in ((1, 10), (8, 32), (64, 10)):
            _same(f"synth-stripe{world}/p{nprobe}k{k}", g.search_batch(q, k, nprobe), full.search_batch(q, k, nprobe))
