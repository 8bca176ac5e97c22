"""List-sharded multi-GPU search.

Inverted lists are independent and a candidate's distance depends only on
(query, its list, its code), so the global top-k of a batch equals the exact
top-k of the union of per-shard top-k lists, ordered by (distance, chunk_id)
(annindex.hpp:54-60, :313). One process per GPU:

  1. every rank holds the entry ranges `prag_gpu_plan_shard_ranges` assigns
     it (whole lists by greedy LPT on list bytes; lists >= 4x the mean size
     striped over all ranks), plus replicated centroids and codebooks, so every rank
     computes the identical probe set (annindex.hpp:277-281);
  2. each rank searches its shard (K1-K4) -> per-shard top-k;
  3. one ncclAllGather of each rank's top-k block, issued by libprag_gpu on
     the search stream (prag_gpu_index_attach_comm; graph-capturable);
  4. every rank runs the exact merge kernel over the gathered blocks.

ShardedIndex is that path. gather_merge below is the same exchange written
with torch.distributed, kept for the CPU (gloo) tests of the host logic.

The reference has no multi-GPU path (it is a single-process scalar library);
this module is the B200 extension the north star asks for. The gather/merge
logic is backend-agnostic so the CPU test suite exercises it over gloo.
"""
from __future__ import annotations

import struct
from typing import Callable, Optional

import numpy as np

from .ivfpq import BatchResult, GpuIndex, merge_topk, plan_shard_ranges, plan_shards

try:
    import torch
    import torch.distributed as dist
except Exception:  # pragma: no cover
    torch = None
    dist = None


def pack_result(r: BatchResult, k: int) -> "torch.Tensor":
    """[nq, 2k+2] int64: ids | distance bits | count | scanned."""
    nq = r.ids.shape[0]
    rec = torch.empty((nq, 2 * k + 2), dtype=torch.int64, device=r.ids.device)
    rec[:, :k] = r.ids
    rec[:, k:2 * k] = r.dist.view(torch.int32).to(torch.int64)
    rec[:, 2 * k] = r.count.to(torch.int64)
    rec[:, 2 * k + 1] = r.scanned
    return rec


def unpack_results(g: "torch.Tensor", k: int):
    """[world, nq, 2k+2] -> ids [world, nq, k], dist, count [world, nq], scanned."""
    ids = g[:, :, :k].contiguous()
    dist_ = g[:, :, k:2 * k].to(torch.int32).view(torch.float32).contiguous()
    cnt = g[:, :, 2 * k].to(torch.int32).contiguous()
    sc = g[:, :, 2 * k + 1].contiguous()
    return ids, dist_, cnt, sc


def gather_merge(local: BatchResult, k: int, merge: Optional[Callable] = None, group=None, root: int = 0):
    """All-gather the per-shard top-k of every rank and merge on `root`.

    `merge(ids, dist, count, scanned, k)` defaults to the GPU merge kernel
    (prag_gpu_merge_topk); returns the merged BatchResult on root, None
    elsewhere."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    rec = pack_result(local, k)
    g = torch.empty((world,) + tuple(rec.shape), dtype=rec.dtype, device=rec.device)
    if rec.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(g, rec, group=group)  # NCCL over NVLink
    else:  # gloo (CPU tests, or a single-GPU functional run of the N>1 path)
        parts = [torch.empty_like(rec, device="cpu") for _ in range(world)]
        dist.all_gather(parts, rec.cpu(), group=group)
        g.copy_(torch.stack(parts))
    if rank != root:
        return None
    ids, dd, cnt, sc = unpack_results(g, k)
    if merge is None:
        return merge_topk(ids, dd, cnt, sc, k, device=ids.device.index or 0,
                          stream=torch.cuda.current_stream(ids.device))
    return merge(ids, dd, cnt, sc, k)


def exchange_unique_id(group=None, src: int = 0) -> bytes:
    """The NCCL unique id (prag_gpu_comm_unique_id on rank `src`), broadcast
    over the torch.distributed group (gloo or nccl): every rank returns the
    same 128 bytes."""
    from .ivfpq import Comm
    obj = [Comm.unique_id() if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id from the broadcast")
    return bytes(uid)


def make_comm(device: int, group=None):
    """prag_gpu_comm of this rank over the group's ranks (collective)."""
    from .ivfpq import Comm
    uid = exchange_unique_id(group)
    return Comm(uid, dist.get_world_size(group), dist.get_rank(group), device)


class ShardedIndex:
    """One rank's shard of a list-sharded index on its own GPU, searched
    collectively through the C ABI: K1-K4 on the rank's lists, one
    ncclAllGather of the per-shard top-k blocks issued by libprag_gpu on the
    search stream, and the exact merge kernel -- every rank gets the merged
    result (prag_gpu_index_attach_comm)."""

    def __init__(self, index: GpuIndex, device: int, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device
        self.index = index
        self.comm = make_comm(device, group)
        index.attach_comm(self.comm)
        self.nlist = index.nlist

    @classmethod
    def load(cls, path: str, device: Optional[int] = None, group=None) -> "ShardedIndex":
        device = torch.cuda.current_device() if device is None else device
        return cls(GpuIndex.load_shard(path, dist.get_rank(group), dist.get_world_size(group), device), device,
                   group)

    @classmethod
    def synthetic(cls, centroids, codewords, ntotal: int, seed: int = 1, sigma: float = 1.0,
                  device: Optional[int] = None, group=None) -> "ShardedIndex":
        device = torch.cuda.current_device() if device is None else device
        ix = GpuIndex.synthetic_shard(centroids, codewords, ntotal, dist.get_rank(group), dist.get_world_size(group),
                                      seed=seed, sigma=sigma, device=device)
        return cls(ix, device, group)

    def search_batch(self, queries, k: int, nprobe: int, stream=None):
        """queries identical on every rank (collective); the merged result."""
        return self.index.search_batch(queries, k, nprobe, stream=stream)

    def plan(self, queries, k: int, nprobe: int, out, stream=None):
        """Captured collective search (graph with the NCCL all-gather)."""
        return self.index.plan(queries, k, nprobe, out, stream=stream)

    def close(self) -> None:
        self.index.attach_comm(None)
        self.index.close()
        self.comm.close()


# ------------------------------------------------------------ shard files
def _read_pragix(path: str):
    """PRAGIX01 (annindex.hpp:335-359) -> (header, centroids, codewords, lists)."""
    with open(path, "rb") as f:
        buf = f.read()
    if buf[:8] != b"PRAGIX01":
        raise ValueError("bad index magic")
    ver, nlist, d, nsq = struct.unpack_from("<IIII", buf, 8)
    off = 24
    cent = np.frombuffer(buf, dtype=np.float32, count=nlist * d, offset=off).reshape(nlist, d)
    off += 4 * nlist * d
    words = np.frombuffer(buf, dtype=np.float32, count=256 * d, offset=off)
    off += 4 * 256 * d
    rec = np.dtype([("id", "<u8"), ("code", "u1", (nsq,))])
    lists = []
    for _ in range(nlist):
        (n,) = struct.unpack_from("<Q", buf, off)
        off += 8
        lists.append(np.frombuffer(buf, dtype=rec, count=n, offset=off))
        off += n * rec.itemsize
    return (ver, nlist, d, nsq), cent, words, lists


def write_shard_pragix(src: str, dst: str, rank: int, world: int) -> np.ndarray:
    """Writes the PRAGIX01 file of one shard: the entry ranges
    plan_shard_ranges gives `rank` (whole lists, or a stripe of a large one;
    others empty), centroids and codebooks replicated. Returns the owner
    array (`world` = striped). Host-only (no GPU)."""
    (ver, nlist, d, nsq), cent, words, lists = _read_pragix(src)
    sizes = [len(l) for l in lists]
    owner = plan_shards(sizes, world)
    beg, end = plan_shard_ranges(sizes, world, rank)
    with open(dst, "wb") as f:
        f.write(b"PRAGIX01")
        f.write(struct.pack("<IIII", ver, nlist, d, nsq))
        f.write(cent.tobytes())
        f.write(words.tobytes())
        for l, b, e in zip(lists, beg, end):
            keep = l[int(b):int(e)]
            f.write(struct.pack("<Q", len(keep)))
            f.write(keep.tobytes())
    return owner
