"""N>1 path on CPU: world_size-2 (and 3) gloo process groups.

Covers the host side of the list-sharded search without a GPU:
LPT shard planning (libprag_gpu.so, host-only), shard PRAGIX01 files, the
packed all-gather of per-shard top-k, and the exact union merge. Each rank's
per-shard top-k comes from the CPU oracle (the checker) reading its shard
file; rank 0 must then reproduce the unsharded oracle result bit-for-bit.
"""
import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_merge(ids, dist, cnt, sc, k):
    import torch
    import _oracle as O
    world, nq, kin = ids.shape
    ids_n = ids.numpy().view(np.uint64)
    dist_n = dist.numpy()
    cnt_n = cnt.numpy().view(np.uint32)
    oi = np.zeros((nq, k), np.uint64)
    od = np.zeros((nq, k), np.float32)
    oc = np.zeros(nq, np.uint32)
    for q in range(nq):
        a, b, c = O.merge_topk(ids_n[:, q], dist_n[:, q], cnt_n[:, q], k)
        oi[q], od[q], oc[q] = a, b, c
    osc = sc.numpy().view(np.uint64).sum(0)
    return oi, od, oc, osc


def _worker(rank, world, port, path, shard_dir, q, nprobe, k, out_dir):
    import torch
    import torch.distributed as dist

    import _oracle as O
    from paper_2403_05676_b200 import distributed as D
    from paper_2403_05676_b200.ivfpq import BatchResult

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        sp = os.path.join(shard_dir, f"shard{rank}of{world}.pragix")
        D.write_shard_pragix(path, sp, rank, world)
        oi = O.OracleIndex(sp)
        ids, dd, cnt, sc = oi.search(q, nprobe, k, threads=1)
        local = BatchResult(torch.from_numpy(ids.view(np.int64)), torch.from_numpy(dd),
                            torch.from_numpy(cnt.view(np.int32)), torch.from_numpy(sc.view(np.int64)))
        merged = D.gather_merge(local, k, merge=_oracle_merge)
        if rank == 0:
            np.savez(os.path.join(out_dir, f"merged{world}.npz"), ids=merged[0], dist=merged[1], count=merged[2],
                     scanned=merged[3])
        else:
            assert merged is None
    finally:
        dist.destroy_process_group()


def _skewed_pragix(src, dst):
    """d384_m32 with list 0 replaced by 4 copies of every entry (new chunk
    ids, same codes): one list far above 4x the mean, so the shard plan
    stripes it, and exact distance ties between entries of different stripes."""
    import struct

    from paper_2403_05676_b200 import distributed as D
    (ver, nlist, d, nsq), cent, words, lists = D._read_pragix(src)
    allent = np.concatenate(lists)
    big = []
    for c in range(4):
        e = allent.copy()
        e["id"] = e["id"] + np.uint64(10**6 * (c + 1))
        big.append(e)
    lists = [np.concatenate(big)] + list(lists[1:])
    with open(dst, "wb") as f:
        f.write(b"PRAGIX01")
        f.write(struct.pack("<IIII", ver, nlist, d, nsq))
        f.write(cent.tobytes())
        f.write(words.tobytes())
        for l in lists:
            f.write(struct.pack("<Q", len(l)))
            f.write(l.tobytes())
    return [len(l) for l in lists]


@pytest.mark.parametrize("world,skew", [(2, False), (3, False), (2, True), (3, True)])
def test_gloo_sharded_search_equals_unsharded(golden, tmp_path, world, skew):
    import torch.multiprocessing as mp

    import _oracle as O
    from paper_2403_05676_b200 import plan_shards
    path, z, grid = golden("d384_m32")
    q = z["queries"]
    nprobe, k = 8, 10
    if skew:
        path = str(tmp_path / "skew.pragix")
        sizes = _skewed_pragix(golden("d384_m32")[0], path)
        assert plan_shards(sizes, world)[0] == world  # list 0 is striped
        nprobe = 32  # every list probed, list 0 included
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, path, str(tmp_path), q, nprobe, k, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    m = np.load(os.path.join(tmp_path, f"merged{world}.npz"))
    ref_ids, ref_dist, ref_cnt, ref_sc = O.OracleIndex(path).search(q, nprobe, k)
    assert (m["count"] == ref_cnt).all()
    assert (m["scanned"] == ref_sc).all()
    for i in range(q.shape[0]):
        c = int(ref_cnt[i])
        assert (m["ids"][i, :c] == ref_ids[i, :c]).all()
        assert (m["dist"][i, :c].view(np.uint32) == ref_dist[i, :c].view(np.uint32)).all()


def test_shard_files_partition_the_index(golden, tmp_path):
    """Every entry lands on exactly one shard (whole lists by LPT, large lists
    striped in rank order); shard sizes follow the plan."""
    from paper_2403_05676_b200 import distributed as D
    path, _, _ = golden("d384_m32")
    _, _, _, lists = D._read_pragix(path)
    sizes = np.array([len(l) for l in lists])
    for world in (2, 3):
        got_lists = [[] for _ in lists]
        loads = []
        for r in range(world):
            sp = str(tmp_path / f"s{world}_{r}.pragix")
            owner = D.write_shard_pragix(path, sp, r, world)
            _, _, _, sl = D._read_pragix(sp)
            got = np.array([len(l) for l in sl])
            assert ((got > 0) <= ((owner == r) | (owner == world))).all()
            loads.append(int(got.sum()))
            for i, l2 in enumerate(sl):
                got_lists[i].append(l2)
        for l, parts in zip(lists, got_lists):  # the stripes concatenate to the list
            cat = np.concatenate(parts)
            assert len(cat) == len(l)
            assert (cat["id"] == l["id"]).all() and (cat["code"] == l["code"]).all()
        assert sum(loads) == int(sizes.sum())
        whole = owner < world
        assert max(loads) <= sizes.sum() / world + (sizes[whole].max() if whole.any() else 0)


def test_pack_unpack_roundtrip():
    import torch
    from paper_2403_05676_b200 import distributed as D
    from paper_2403_05676_b200.ivfpq import BatchResult
    rng = np.random.default_rng(0)
    nq, k = 5, 4
    r = BatchResult(torch.from_numpy(rng.integers(0, 2**62, (nq, k), dtype=np.int64)),
                    torch.from_numpy(rng.random((nq, k), dtype=np.float32) * 1e3),
                    torch.from_numpy(rng.integers(0, k + 1, nq).astype(np.int32)),
                    torch.from_numpy(rng.integers(0, 2**40, nq, dtype=np.int64)))
    g = D.pack_result(r, k)[None]
    ids, dd, cnt, sc = D.unpack_results(g, k)
    assert torch.equal(ids[0], r.ids) and torch.equal(cnt[0], r.count) and torch.equal(sc[0], r.scanned)
    assert torch.equal(dd[0].view(torch.int32), r.dist.view(torch.int32))


def _uid_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import paper_2403_05676_b200 as pg
    from paper_2403_05676_b200 import distributed as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        uid = D.exchange_unique_id()
        with open(os.path.join(out_dir, f"uid{rank}.bin"), "wb") as f:
            f.write(uid)
        # no GPU here: the communicator itself must refuse, not fall back
        if pg.device_count() == 0:
            try:
                pg.Comm(uid, world, rank, 0)
                raise AssertionError("comm_init without a device must fail")
            except pg.NoDeviceError:
                pass
    finally:
        dist.destroy_process_group()


def test_gloo_world2_nccl_unique_id_rendezvous(tmp_path):
    """The host side of the distributed shard (ShardedIndex / bench.py
    --gpus N): rank 0's prag_gpu_comm_unique_id reaches every rank intact
    over a world-2 gloo group."""
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_uid_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    a = open(tmp_path / "uid0.bin", "rb").read()
    b = open(tmp_path / "uid1.bin", "rb").read()
    assert len(a) == 128 and a == b and any(a)
