"""Python mirror of the reference retrieval API over the B200 C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/prag/annindex.hpp:35-50, :262-315 and
perfmodel.hpp:19-26, :92-157), so the parity tests read like the reference's
own tests (test_annindex.cpp, test_perfmodel.cpp). Compute happens only in
libprag_gpu.so (hand-written sm_100a kernels); this module moves pointers.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Callable, Iterable, List, Optional, Sequence

import numpy as np

from ._lib import (ConfigError, FormatError, IndexDesc, MEASURE_FN, PerfModelC, Timings, TrainParamsC, check, lib)

try:  # torch is plumbing only (device buffers / streams); optional here
    import torch
except Exception:  # pragma: no cover
    torch = None


# ------------------------------------------------------------------ types
@dataclass
class SearchParams:
    """annindex.hpp:35-39."""
    nprobe: int = 1
    k: int = 2
    exact_rerank: bool = False


@dataclass
class ScoredId:
    """annindex.hpp:41-44."""
    chunk_id: int = 0
    distance: float = 0.0


@dataclass
class SearchResult:
    """annindex.hpp:46-50: ascending distance, ties by lower id."""
    neighbors: List[ScoredId] = field(default_factory=list)
    scanned_vectors: int = 0
    scanned_lists: int = 0


@dataclass
class BatchResult:
    ids: object        # [nq, k] uint64 (numpy) / int64 view (torch)
    dist: object       # [nq, k] float32
    count: object      # [nq] uint32 / int32
    scanned: object    # [nq] uint64 / int64

    def result(self, q: int, nprobe: int) -> SearchResult:
        ids = np.asarray(_to_numpy(self.ids))
        dist = np.asarray(_to_numpy(self.dist))
        c = int(np.asarray(_to_numpy(self.count))[q])
        return SearchResult([ScoredId(int(ids[q, i]), float(dist[q, i])) for i in range(c)],
                            int(np.asarray(_to_numpy(self.scanned))[q]), nprobe)


def _to_numpy(a):
    if torch is not None and isinstance(a, torch.Tensor):
        t = a.detach().cpu()
        if t.dtype == torch.int64:
            return t.numpy().view(np.uint64)
        if t.dtype == torch.int32:
            return t.numpy().view(np.uint32)
        return t.numpy()
    return a


def _ptr(a) -> C.c_void_p:
    if a is None:
        return C.c_void_p(0)
    if torch is not None and isinstance(a, torch.Tensor):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def _stream_ptr(stream) -> C.c_void_p:
    if stream is None:
        return C.c_void_p(0)
    if torch is not None and isinstance(stream, torch.cuda.Stream):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def device_count() -> int:
    return lib().prag_gpu_device_count()


# ------------------------------------------------------------------ index
class GpuIndex:
    """HBM-resident IVF-PQ index (replaces the IvfIndex + PqCodebook pair)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        d = IndexDesc()
        check(lib().prag_gpu_index_describe(self._h, C.byref(d)))
        self.desc = d
        self.nlist, self.d, self.nsq, self.sub_dim = d.nlist, d.d, d.nsq, d.sub_dim
        self.ntotal, self.device = d.ntotal, d.device

    # constructors ------------------------------------------------------
    @classmethod
    def load(cls, path: str, device: int = 0) -> "GpuIndex":
        """prag::load_index (annindex.hpp:361-411) straight into HBM."""
        h = C.c_void_p()
        check(lib().prag_gpu_index_load(str(path).encode(), device, C.byref(h)))
        return cls(h)

    @classmethod
    def load_shard(cls, path: str, rank: int, world: int, device: int = 0) -> "GpuIndex":
        h = C.c_void_p()
        check(lib().prag_gpu_index_load_shard(str(path).encode(), device, rank, world, C.byref(h)))
        return cls(h)

    @classmethod
    def from_host(cls, centroids, codewords, list_off, ids, codes, device: int = 0) -> "GpuIndex":
        centroids = np.ascontiguousarray(centroids, dtype=np.float32)
        codewords = np.ascontiguousarray(codewords, dtype=np.float32)
        list_off = np.ascontiguousarray(list_off, dtype=np.uint64)
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        nlist, d = centroids.shape
        nsq = codewords.shape[0]
        h = C.c_void_p()
        check(lib().prag_gpu_index_from_host(nlist, d, nsq, _ptr(centroids), _ptr(codewords), _ptr(list_off),
                                             _ptr(ids), _ptr(codes), device, C.byref(h)))
        return cls(h)

    @classmethod
    def synthetic(cls, centroids, codewords, ntotal: int, seed: int = 1, sigma: float = 1.0,
                  device: int = 0) -> "GpuIndex":
        """Config-D fixture built in HBM (prag_gpu_index_synthetic; k <= 32)."""
        centroids = np.ascontiguousarray(centroids, dtype=np.float32)
        codewords = np.ascontiguousarray(codewords, dtype=np.float32)
        nlist, d = centroids.shape
        nsq = codewords.shape[0]
        h = C.c_void_p()
        check(lib().prag_gpu_index_synthetic(nlist, d, nsq, ntotal, seed, sigma, _ptr(centroids), _ptr(codewords),
                                             device, C.byref(h)))
        return cls(h)

    @classmethod
    def synthetic_shard(cls, centroids, codewords, ntotal: int, rank: int, world: int, seed: int = 1,
                        sigma: float = 1.0, device: int = 0) -> "GpuIndex":
        """Rank `rank` of `world` of the synthetic index (same entries, ids and
        codes as GpuIndex.synthetic with the same arguments)."""
        centroids = np.ascontiguousarray(centroids, dtype=np.float32)
        codewords = np.ascontiguousarray(codewords, dtype=np.float32)
        nlist, d = centroids.shape
        nsq = codewords.shape[0]
        h = C.c_void_p()
        check(lib().prag_gpu_index_synthetic_shard(nlist, d, nsq, ntotal, seed, sigma, _ptr(centroids),
                                                   _ptr(codewords), rank, world, device, C.byref(h)))
        return cls(h)

    @classmethod
    def load_sharded(cls, path: str, devices: Sequence[int]) -> "GpuIndex":
        """One process, several GPUs: the index's lists spread over `devices`
        (LPT on bytes; devices may repeat). Searches run every shard on its own
        device and merge on devices[0] reading the shards over NVLink."""
        dv = np.ascontiguousarray(devices, dtype=np.int32)
        h = C.c_void_p()
        check(lib().prag_gpu_index_load_sharded(str(path).encode(), _ptr(dv), len(dv), C.byref(h)))
        return cls(h)

    @classmethod
    def group(cls, shards: Sequence["GpuIndex"]) -> "GpuIndex":
        """Group handle over shard handles (ranks 0..n-1 of world n); takes
        ownership of them."""
        arr = (C.c_void_p * len(shards))(*[s._h for s in shards])
        h = C.c_void_p()
        check(lib().prag_gpu_index_group(arr, len(shards), C.byref(h)))
        for s in shards:
            s._h = None  # owned by the group now
        return cls(h)

    def attach_comm(self, comm: Optional["Comm"]) -> None:
        """Makes searches on this shard collective over `comm` (NCCL):
        every rank passes the same queries and gets the merged result."""
        check(lib().prag_gpu_index_attach_comm(self._h, comm._h if comm is not None else None))
        self._comm = comm

    def store(self, path: str) -> None:
        """prag::store_index (annindex.hpp:335-359) of the resident index."""
        check(lib().prag_gpu_index_store(self._h, str(path).encode()))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().prag_gpu_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # queries -------------------------------------------------------------
    def list_sizes(self) -> np.ndarray:
        out = np.zeros(self.nlist, dtype=np.uint64)
        check(lib().prag_gpu_index_list_sizes(self._h, _ptr(out)))
        return out

    def set_embeddings(self, embeddings) -> None:
        """Raw embeddings [n, d] (indexed by chunk id) for exact rerank
        (annindex.hpp:307-312); None detaches."""
        if embeddings is None:
            check(lib().prag_gpu_index_set_embeddings(self._h, None, 0))
            self._emb_key = None
            return
        if torch is not None and isinstance(embeddings, torch.Tensor) and embeddings.is_cuda:
            e = embeddings.contiguous()
            n = e.shape[0]
        else:
            e = np.ascontiguousarray(embeddings, dtype=np.float32).reshape(-1, self.d)
            n = e.shape[0]
        check(lib().prag_gpu_index_set_embeddings(self._h, _ptr(e), n))
        self._emb_key = id(embeddings)

    def search_batch(self, queries, k: int, nprobe: int, stream=None, out: Optional[BatchResult] = None,
                     exact_rerank: bool = False) -> BatchResult:
        """Batch prag::search: queries [nq, d] float32, host (numpy / CPU tensor)
        or device (CUDA tensor). Device queries -> device outputs, asynchronous
        on `stream` (default: torch's current stream). exact_rerank uses the
        embeddings given to set_embeddings()."""
        on_dev = torch is not None and isinstance(queries, torch.Tensor) and queries.is_cuda
        if on_dev:
            q = queries.contiguous()
            if q.dtype != torch.float32:
                raise ConfigError("queries must be float32")
            self._check_dev_queries(q)
            nq = q.shape[0] if q.dim() == 2 else 1
            if out is None:
                out = BatchResult(torch.empty((nq, k), dtype=torch.int64, device=q.device),
                                  torch.empty((nq, k), dtype=torch.float32, device=q.device),
                                  torch.empty((nq,), dtype=torch.int32, device=q.device),
                                  torch.empty((nq,), dtype=torch.int64, device=q.device))
            if stream is None:
                stream = torch.cuda.current_stream(q.device)
        else:
            if torch is not None and isinstance(queries, torch.Tensor):
                queries = queries.numpy()
            q = np.ascontiguousarray(queries, dtype=np.float32).reshape(-1, self.d)
            nq = q.shape[0]
            if out is None:
                out = BatchResult(np.zeros((nq, k), dtype=np.uint64), np.zeros((nq, k), dtype=np.float32),
                                  np.zeros(nq, dtype=np.uint32), np.zeros(nq, dtype=np.uint64))
        if (not on_dev) and q.shape[1] != self.d:
            raise ConfigError(f"query dimension {q.shape[1]} != index d {self.d}")
        all_dev = on_dev and all(torch is not None and isinstance(x, torch.Tensor) and x.is_cuda
                                 for x in (out.ids, out.dist, out.count, out.scanned))
        if exact_rerank:
            fn = lib().prag_gpu_search_rerank
        else:
            fn = lib().prag_gpu_search_device if all_dev else lib().prag_gpu_search
        check(fn(self._h, _ptr(q), nq, nprobe, k, _ptr(out.ids), _ptr(out.dist), _ptr(out.count),
                 _ptr(out.scanned), _stream_ptr(stream)))
        return out

    def _check_dev_queries(self, q) -> None:
        # the C ABI takes no d: a device tensor of the wrong width would be
        # read as nq x d floats out of bounds
        if q.dim() not in (1, 2) or q.shape[-1] != self.d:
            raise ConfigError(f"queries must be [nq, {self.d}] (or [{self.d}]), got {tuple(q.shape)}")

    def plan(self, queries, k: int, nprobe: int, out: BatchResult, stream=None) -> "SearchPlan":
        """A captured search (prag_gpu_plan_create) over fixed CUDA buffers:
        write new queries into `queries`, then SearchPlan.launch()."""
        if not (torch is not None and isinstance(queries, torch.Tensor) and queries.is_cuda):
            raise ConfigError("plan: queries must be a CUDA tensor")
        if queries.dtype != torch.float32 or not queries.is_contiguous():
            raise ConfigError("plan: queries must be a contiguous float32 tensor")
        self._check_dev_queries(queries)
        h = C.c_void_p()
        nq = queries.shape[0] if queries.dim() == 2 else 1
        check(lib().prag_gpu_plan_create(self._h, _ptr(queries), nq, nprobe, k, _ptr(out.ids), _ptr(out.dist),
                                         _ptr(out.count), _ptr(out.scanned), _stream_ptr(stream), C.byref(h)))
        return SearchPlan(h, self, queries, out)

    def probe(self, queries, nprobe: int):
        """Coarse quantizer only (annindex.hpp:277-281)."""
        q = np.ascontiguousarray(queries, dtype=np.float32).reshape(-1, self.d)
        lists = np.zeros((q.shape[0], nprobe), dtype=np.uint32)
        dist = np.zeros((q.shape[0], nprobe), dtype=np.float32)
        check(lib().prag_gpu_probe(self._h, _ptr(q), q.shape[0], nprobe, _ptr(lists), _ptr(dist), None))
        return lists, dist

    def set_sm_budget(self, sms: int) -> None:
        """Persistent search grids on at most `sms` SMs (0 = all): retrieval
        beside work pinned to the other SMs (prag_gpu_set_sm_budget)."""
        check(lib().prag_gpu_set_sm_budget(self._h, int(sms)))

    def set_scan_path(self, path: int) -> None:
        """0 = automatic (fast lane-skewed path when eligible), 1 = generic."""
        check(lib().prag_gpu_set_scan_path(self._h, path))

    def set_coarse_path(self, path: int) -> None:
        """0 = automatic (tensor-core pre-filter + exact window), 1 = exact SIMT."""
        check(lib().prag_gpu_set_coarse_path(self._h, path))

    # profiling -------------------------------------------------------------
    def set_profiling(self, on: bool) -> None:
        check(lib().prag_gpu_set_profiling(self._h, 1 if on else 0))

    def last_timings(self) -> dict:
        t = Timings()
        check(lib().prag_gpu_last_timings(self._h, C.byref(t)))
        return {f: getattr(t, f) for f, _ in Timings._fields_}


class Comm:
    """NCCL communicator of one rank (prag_gpu_comm_*): the exchange step of
    a distributed list-sharded index."""

    def __init__(self, unique_id: bytes, world: int, rank: int, device: int):
        if len(unique_id) != 128:
            raise ConfigError("unique id must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        check(lib().prag_gpu_comm_init(buf, world, rank, device, C.byref(h)))
        self._h, self.world, self.rank, self.device = h, world, rank, device

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().prag_gpu_comm_unique_id(buf))
        return bytes(buf)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().prag_gpu_comm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SearchPlan:
    """CUDA-graph replay of one search shape over fixed device buffers."""

    def __init__(self, handle, index, queries, out):
        self._h, self._index, self.queries, self.out = handle, index, queries, out

    def launch(self, stream=None) -> BatchResult:
        check(lib().prag_gpu_plan_launch(self._h, _stream_ptr(stream)))
        return self.out

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().prag_gpu_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GpuChunkEmbedder:
    """Device-resident prag::ChunkEmbedder (tokendb.hpp:84-124): bit-identical
    bag-of-tokens embeddings, computed on the GPU."""

    def __init__(self, d: int, seed: int, vocab: int = 257, device: int = 0):
        h = C.c_void_p()
        check(lib().prag_gpu_embedder_create(d, seed, vocab, device, C.byref(h)))
        self._h, self.d, self.seed, self.vocab = h, d, seed, vocab

    def embed(self, chunks, stream=None):
        """chunks: [n, m] token ids (numpy / CUDA tensor) -> [n, d] float32."""
        on_dev = torch is not None and isinstance(chunks, torch.Tensor) and chunks.is_cuda
        if on_dev:
            t = chunks.contiguous().to(torch.int32)
            n, m = t.shape
            out = torch.empty((n, self.d), dtype=torch.float32, device=t.device)
            if stream is None:
                stream = torch.cuda.current_stream(t.device)
        else:
            t = np.ascontiguousarray(chunks, dtype=np.uint32)
            if t.ndim == 1:
                t = t.reshape(1, -1)
            n, m = t.shape
            out = np.zeros((n, self.d), dtype=np.float32)
        check(lib().prag_gpu_embed(self._h, _ptr(t), n, m, _ptr(out), _stream_ptr(stream)))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().prag_gpu_embedder_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ build
@dataclass
class TrainParams:
    """annindex.hpp:152-160 (same defaults)."""
    nlist: int = 64
    n_subquantizers: int = 0          # 0 -> d / 4
    seed: int = 7
    kmeans_iterations: int = 25
    train_sample_cap: int = 32768


@dataclass
class TrainedIndex:
    """prag::train_index's {IvfIndex, PqCodebook} in flattened list-major form:
    centroids [nlist][d], codewords [nsq][256][d/nsq], list_off [nlist+1],
    ids [n] (vector indices, each list in vector order), codes [n][nsq]."""
    centroids: np.ndarray
    codewords: np.ndarray
    list_off: np.ndarray
    ids: np.ndarray
    codes: np.ndarray

    def to_gpu(self, device: int = 0) -> "GpuIndex":
        return GpuIndex.from_host(self.centroids, self.codewords, self.list_off, self.ids, self.codes, device)

    def write_pragix(self, path: str) -> None:
        """prag::store_index (annindex.hpp:335-359)."""
        from .fixtures import write_pragix
        write_pragix(path, self.centroids, self.codewords, self.list_off, self.ids, self.codes)


def train_index(vectors, params: Optional[TrainParams] = None, device: int = 0) -> TrainedIndex:
    """prag::train_index (annindex.hpp:164-241) on the device, bit-exact
    (prag_gpu_train_index). `vectors`: n x d fp32 (numpy or a CUDA tensor)."""
    p = params or TrainParams()
    if torch is not None and isinstance(vectors, torch.Tensor):
        if vectors.dtype != torch.float32 or vectors.dim() != 2:
            raise ConfigError("train_index: vectors must be a 2-D float32 tensor")
        vectors = vectors.contiguous()
        n, d = vectors.shape
    else:
        vectors = np.ascontiguousarray(vectors, dtype=np.float32)
        if vectors.ndim != 2:
            raise ConfigError("train_index: vectors must be n x d")
        n, d = vectors.shape
    nsq = p.n_subquantizers if p.n_subquantizers else max(1, d // 4)
    nlist = p.nlist
    ok = n > 0 and d > 0 and 0 < nlist <= n and d % nsq == 0
    shp = (max(nlist, 1), max(d, 1))
    cents = np.zeros(shp, dtype=np.float32)
    words = np.zeros((nsq, 256, max(d // nsq, 1)) if ok else (1,), dtype=np.float32)
    off = np.zeros(max(nlist, 0) + 1, dtype=np.uint64)
    ids = np.zeros(max(n, 1), dtype=np.uint64)
    codes = np.zeros((max(n, 1), nsq), dtype=np.uint8)
    c = TrainParamsC(nlist, p.n_subquantizers, p.seed, p.kmeans_iterations, 0, p.train_sample_cap)
    check(lib().prag_gpu_train_index(_ptr(vectors) if n else None, n, d, C.byref(c), device, _ptr(cents),
                                     _ptr(words), _ptr(off), _ptr(ids), _ptr(codes)))
    return TrainedIndex(cents, words, off, ids[:n], codes[:n])


def load_index(path: str, device: int = 0) -> GpuIndex:
    return GpuIndex.load(path, device)


def search(index: GpuIndex, query, params: SearchParams, embeddings=None) -> SearchResult:
    """prag::search (annindex.hpp:262-315) for one query."""
    if params.exact_rerank:
        if embeddings is None:  # annindex.hpp:269-271
            raise ConfigError("search: exact_rerank requires raw embeddings")
        if getattr(index, "_emb_key", None) != id(embeddings):
            index.set_embeddings(embeddings)
    r = index.search_batch(np.asarray(query, dtype=np.float32).reshape(1, -1), params.k, params.nprobe,
                           exact_rerank=params.exact_rerank)
    return r.result(0, params.nprobe)


def brute_force_search(vectors, queries, k: int, device: int = 0) -> BatchResult:
    """prag::brute_force_search (annindex.hpp:244-257) for a batch, on the
    device: exact top-k by full-precision squared L2, ties by lower row id."""
    v = np.ascontiguousarray(vectors, dtype=np.float32)
    q = np.ascontiguousarray(queries, dtype=np.float32).reshape(-1, v.shape[1])
    nq = q.shape[0]
    out = BatchResult(np.zeros((nq, k), dtype=np.uint64), np.zeros((nq, k), dtype=np.float32),
                      np.zeros(nq, dtype=np.uint32), np.full(nq, v.shape[0], dtype=np.uint64))
    check(lib().prag_gpu_brute_force(_ptr(v), v.shape[0], v.shape[1], _ptr(q), nq, k, device, _ptr(out.ids),
                                     _ptr(out.dist), _ptr(out.count)))
    return out


def recall_at_k(approx: SearchResult, exact: SearchResult) -> float:
    """annindex.hpp:317-327: |approx ∩ exact| / |exact| over chunk ids (1.0 if exact is empty)."""
    if not exact.neighbors:
        return 1.0
    got = {n.chunk_id for n in approx.neighbors}
    return sum(1 for e in exact.neighbors if e.chunk_id in got) / len(exact.neighbors)


# ------------------------------------------------------------ multi-GPU
def plan_shards(list_sizes: Sequence[int], world: int) -> np.ndarray:
    """Owner rank of every list; `world` marks a list striped over all ranks."""
    s = np.ascontiguousarray(list_sizes, dtype=np.uint64)
    owner = np.zeros(len(s), dtype=np.uint32)
    check(lib().prag_gpu_plan_shards(_ptr(s), len(s), world, _ptr(owner)))
    return owner


def plan_shard_ranges(list_sizes: Sequence[int], world: int, rank: int):
    """(begin, end) entry range of every list on shard `rank` (whole lists or stripes)."""
    s = np.ascontiguousarray(list_sizes, dtype=np.uint64)
    b = np.zeros(len(s), dtype=np.uint64)
    e = np.zeros(len(s), dtype=np.uint64)
    check(lib().prag_gpu_plan_shard_ranges(_ptr(s), len(s), world, rank, _ptr(b), _ptr(e)))
    return b, e


def merge_topk(ids, dist, count, scanned, k: int, device: int = 0, stream=None, out=None):
    """K5: exact top-k of the union of per-shard results.
    ids/dist [nparts, nq, kin], count/scanned [nparts, nq]; numpy or CUDA tensors."""
    on_dev = torch is not None and isinstance(ids, torch.Tensor) and ids.is_cuda
    nparts, nq, kin = ids.shape
    if out is None:
        if on_dev:
            out = BatchResult(torch.empty((nq, k), dtype=torch.int64, device=ids.device),
                              torch.empty((nq, k), dtype=torch.float32, device=ids.device),
                              torch.empty((nq,), dtype=torch.int32, device=ids.device),
                              torch.empty((nq,), dtype=torch.int64, device=ids.device))
        else:
            ids = np.ascontiguousarray(ids, dtype=np.uint64)
            dist = np.ascontiguousarray(dist, dtype=np.float32)
            count = np.ascontiguousarray(count, dtype=np.uint32)
            scanned = None if scanned is None else np.ascontiguousarray(scanned, dtype=np.uint64)
            out = BatchResult(np.zeros((nq, k), dtype=np.uint64), np.zeros((nq, k), dtype=np.float32),
                              np.zeros(nq, dtype=np.uint32), np.zeros(nq, dtype=np.uint64))
    if on_dev and stream is None:
        stream = torch.cuda.current_stream(ids.device)
    check(lib().prag_gpu_merge_topk(_ptr(ids), _ptr(dist), _ptr(count), _ptr(scanned), nparts, nq, kin, k,
                                    _ptr(out.ids), _ptr(out.dist), _ptr(out.count), _ptr(out.scanned), device,
                                    _stream_ptr(stream)))
    return out


# ------------------------------------------------------ performance model
@dataclass
class RetrievalPerfModel:
    """perfmodel.hpp:19-26."""
    slope_s: float = 0.0
    intercept_s: float = 0.0
    fit_residual_s: float = 0.0
    clamped: bool = False

    def predict(self, nprobe: int) -> float:
        return self.slope_s * nprobe + self.intercept_s

    def _c(self) -> PerfModelC:
        return PerfModelC(self.slope_s, self.intercept_s, self.fit_residual_s, int(self.clamped), 0)

    @classmethod
    def _from_c(cls, m: PerfModelC) -> "RetrievalPerfModel":
        return cls(m.slope_s, m.intercept_s, m.fit_residual_s, bool(m.clamped))


def calibrate_retrieval(retrieve: Callable[[int], float], nprobe_grid: Iterable[int], repeats: int = 5,
                        warmups: int = 2) -> RetrievalPerfModel:
    """perfmodel.hpp:92-117 over a caller-supplied timer (its std::function hook)."""
    grid = np.ascontiguousarray(list(nprobe_grid), dtype=np.uint32)
    errors = []

    def cb(nprobe, _ctx):
        try:
            return float(retrieve(int(nprobe)))
        except Exception as e:  # surface Python errors after the C call returns
            errors.append(e)
            return 0.0

    fn = MEASURE_FN(cb)
    m = PerfModelC()
    check(lib().prag_gpu_calibrate_with(fn, None, _ptr(grid), len(grid), repeats, warmups, C.byref(m)))
    if errors:
        raise errors[0]
    return RetrievalPerfModel._from_c(m)


def calibrate_gpu(index: GpuIndex, queries, k: int, nprobe_grid: Iterable[int], repeats: int = 5,
                  warmups: int = 2):
    """calibrate_retrieval fed with the GPU batch-latency curve (host queries in,
    host results out, wall clock per batch). Returns (model, {nprobe: median_s})."""
    q = np.ascontiguousarray(queries, dtype=np.float32).reshape(-1, index.d)
    grid = np.ascontiguousarray(list(nprobe_grid), dtype=np.uint32)
    uniq = np.unique(grid)
    lat = np.zeros(max(1, len(uniq)), dtype=np.float64)
    m = PerfModelC()
    check(lib().prag_gpu_calibrate_retrieval(index._h, _ptr(q), q.shape[0], k, _ptr(grid), len(grid), repeats,
                                             warmups, C.byref(m), _ptr(lat)))
    return RetrievalPerfModel._from_c(m), {int(n): float(t) for n, t in zip(uniq, lat)}


def select_nprobe(model: RetrievalPerfModel, budget_s: float, nlist: int, safety_margin: float = 0.10) -> int:
    """perfmodel.hpp:148-157."""
    m = model._c()
    return int(lib().prag_gpu_select_nprobe(C.byref(m), budget_s, nlist, safety_margin))


def store_perf_model(model: RetrievalPerfModel, path: str, inference_buckets=()) -> None:
    """Same JSON schema as perfmodel.hpp:190-202 (clamped is not serialised)."""
    j = {"slope_s": model.slope_s, "intercept_s": model.intercept_s, "fit_residual_s": model.fit_residual_s,
         "inference_buckets": [dict(b) for b in inference_buckets]}
    with open(path, "w") as f:
        f.write(json.dumps(j, indent=2) + "\n")


def load_perf_model(path: str) -> RetrievalPerfModel:
    """perfmodel.hpp:204-223 (retrieval part)."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise FormatError("cannot open for reading: " + path)
    except json.JSONDecodeError as e:
        raise FormatError(f"invalid perf model JSON in {path}: {e}")
    return RetrievalPerfModel(float(j["slope_s"]), float(j["intercept_s"]), float(j["fit_residual_s"]))
