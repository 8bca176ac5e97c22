"""ctypes bindings to the CPU oracle (oracle/liboracle.so) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker. The oracle restates
/root/reference/proj/include/prag/annindex.hpp:262-315 op-for-op (see
oracle/prag_oracle.c); it is pinned to the reference through tests/golden/.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
import subprocess

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(REPO, "oracle", "liboracle.so")
REF_TOOL = os.path.join(REPO, "oracle", "_ref", "ref_tool")

_lib = None


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        L = C.CDLL(ORACLE_SO)
        P = C.c_void_p
        L.ora_last_error.restype = C.c_char_p
        L.ora_load_index.argtypes = [C.c_char_p, C.POINTER(P)]
        L.ora_free_index.argtypes = [P]
        L.ora_squared_l2.argtypes = [P, P, C.c_size_t]
        L.ora_squared_l2.restype = C.c_float
        L.ora_search.argtypes = [P, P, C.c_uint32, C.c_uint32, P, P, P, P, P]
        L.ora_search_batch.argtypes = [P, P, C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, C.c_int]
        L.ora_probe_lists.argtypes = [P, P, C.c_uint32, P, P]
        L.ora_brute_force.argtypes = [P, C.c_uint64, C.c_uint32, P, C.c_uint32, P, P, P]
        L.ora_merge_topk.argtypes = [P, P, P, C.c_uint32, C.c_uint32, C.c_uint32, P, P, P]
        L.ora_least_squares.argtypes = [P, P, C.c_size_t, P, P, P, P]
        L.ora_median.argtypes = [P, C.c_size_t]
        L.ora_median.restype = C.c_double
        L.ora_select_nprobe.argtypes = [C.c_double, C.c_double, C.c_double, C.c_uint32, C.c_double]
        L.ora_select_nprobe.restype = C.c_uint32
        L.ora_splitmix_next.argtypes = [P]
        L.ora_splitmix_next.restype = C.c_uint64
        L.ora_splitmix_gaussian.argtypes = [P]
        L.ora_splitmix_gaussian.restype = C.c_double
        L.ora_hash_combine.argtypes = [C.c_uint64, C.c_uint64]
        L.ora_hash_combine.restype = C.c_uint64
        L.ora_random_vectors.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, P]
        L.ora_train_index.argtypes = [P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int,
                                      C.c_uint64, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class SplitMix64:
    """common.hpp:33-64 through the oracle's C restatement (same libm)."""

    def __init__(self, seed: int):
        self.state = C.c_uint64(seed)

    def next_u64(self) -> int:
        return lib().ora_splitmix_next(C.byref(self.state))

    def next_below(self, bound: int) -> int:
        return self.next_u64() % bound

    def next_gaussian(self) -> float:
        return lib().ora_splitmix_gaussian(C.byref(self.state))


def random_vectors(n: int, d: int, seed: int) -> np.ndarray:
    """test_annindex.cpp:12-19 recipe."""
    out = np.empty((n, d), dtype=np.float32)
    lib().ora_random_vectors(seed, n, d, _p(out))
    return out


def train_index(v: np.ndarray, nlist: int, nsq: int = 0, seed: int = 7, iters: int = 25, cap: int = 32768):
    """annindex.hpp:164-241 via the C restatement: (centroids, codewords,
    list_off, ids, codes), flattened list-major."""
    v = np.ascontiguousarray(v, dtype=np.float32)
    n, d = v.shape
    m = nsq if nsq else max(1, d // 4)
    cents = np.zeros((max(nlist, 1), d), np.float32)
    words = np.zeros((m, 256, max(d // m, 1)), np.float32)
    off = np.zeros(nlist + 1, np.uint64)
    ids = np.zeros(max(n, 1), np.uint64)
    codes = np.zeros((max(n, 1), m), np.uint8)
    rc = lib().ora_train_index(_p(v), n, d, nlist, nsq, seed, iters, cap, _p(cents), _p(words), _p(off), _p(ids),
                               _p(codes))
    if rc:
        raise OracleError(rc, lib().ora_last_error().decode())
    return cents, words, off, ids[:n], codes[:n]


def noisy_queries(base: np.ndarray, nq: int, seed: int, scale: float) -> np.ndarray:
    """annindex_main.cpp:66-74 recipe: a DB row plus scale*N(0,1) noise, in fp32."""
    rng = SplitMix64(seed)
    q = np.empty((nq, base.shape[1]), dtype=np.float32)
    s = np.float32(scale)
    for i in range(nq):
        v = base[rng.next_below(base.shape[0])].copy()
        for j in range(v.shape[0]):
            v[j] = np.float32(v[j] + np.float32(s * np.float32(rng.next_gaussian())))
        q[i] = v
    return q


class OracleIndex:
    def __init__(self, path: str):
        h = C.c_void_p()
        rc = lib().ora_load_index(path.encode(), C.byref(h))
        if rc:
            raise OracleError(rc, lib().ora_last_error().decode())
        self.h = h
        hdr = C.cast(h, C.POINTER(C.c_uint32))
        self.nlist, self.d, self.nsq, self.sub_dim = hdr[0], hdr[1], hdr[2], hdr[3]

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ora_free_index(self.h)
                self.h = None
        except Exception:
            pass

    def search(self, queries: np.ndarray, nprobe: int, k: int, threads: int = 0):
        q = np.ascontiguousarray(queries, dtype=np.float32).reshape(-1, self.d)
        nq = q.shape[0]
        ids = np.zeros((nq, k), dtype=np.uint64)
        dist = np.zeros((nq, k), dtype=np.float32)
        count = np.zeros(nq, dtype=np.uint32)
        scanned = np.zeros(nq, dtype=np.uint64)
        if threads <= 0:
            threads = min(os.cpu_count() or 1, max(1, nq))
        rc = lib().ora_search_batch(self.h, _p(q), nq, nprobe, k, _p(ids), _p(dist), _p(count),
                                    _p(scanned), threads)
        if rc:
            raise OracleError(rc, lib().ora_last_error().decode())
        return ids, dist, count, scanned

    def probe_lists(self, query: np.ndarray, nprobe: int):
        q = np.ascontiguousarray(query, dtype=np.float32)
        lists = np.zeros(nprobe, dtype=np.uint32)
        dist = np.zeros(nprobe, dtype=np.float32)
        rc = lib().ora_probe_lists(self.h, _p(q), nprobe, _p(lists), _p(dist))
        if rc:
            raise OracleError(rc, lib().ora_last_error().decode())
        return lists, dist


def merge_topk(ids: np.ndarray, dist: np.ndarray, count: np.ndarray, k: int):
    """ids/dist: [nparts][kin]; returns exact top-k of the union."""
    ids = np.ascontiguousarray(ids, dtype=np.uint64)
    dist = np.ascontiguousarray(dist, dtype=np.float32)
    count = np.ascontiguousarray(count, dtype=np.uint32)
    nparts, kin = ids.shape
    oi = np.zeros(k, dtype=np.uint64)
    od = np.zeros(k, dtype=np.float32)
    oc = np.zeros(1, dtype=np.uint32)
    lib().ora_merge_topk(_p(ids), _p(dist), _p(count), nparts, kin, k, _p(oi), _p(od), _p(oc))
    return oi, od, int(oc[0])


def select_nprobe(slope_s, intercept_s, budget_s, nlist, margin=0.10) -> int:
    return lib().ora_select_nprobe(slope_s, intercept_s, budget_s, nlist, margin)


def least_squares(x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(4, dtype=np.float64)
    lib().ora_least_squares(_p(x), _p(y), len(x), C.c_void_p(out.ctypes.data),
                            C.c_void_p(out.ctypes.data + 8), C.c_void_p(out.ctypes.data + 16),
                            C.c_void_p(out.ctypes.data + 24))
    return tuple(out)


# ---------------------------------------------------------------- PRAGIX01 I/O
def write_pragix(path, centroids, codewords, lists):
    """PRAGIX01 writer (format of annindex.hpp:335-359).

    centroids [nlist][d] f32, codewords [nsq][256][sub_dim] f32,
    lists: sequence of (ids u64[n], codes u8[n][nsq]).
    """
    centroids = np.ascontiguousarray(centroids, dtype=np.float32)
    codewords = np.ascontiguousarray(codewords, dtype=np.float32)
    nlist, d = centroids.shape
    nsq = codewords.shape[0]
    with open(path, "wb") as f:
        f.write(b"PRAGIX01")
        f.write(struct.pack("<IIII", 1, nlist, d, nsq))
        f.write(centroids.tobytes())
        f.write(codewords.tobytes())
        for ids, codes in lists:
            ids = np.asarray(ids, dtype=np.uint64)
            codes = np.asarray(codes, dtype=np.uint8).reshape(len(ids), nsq)
            f.write(struct.pack("<Q", len(ids)))
            rec = np.zeros(len(ids), dtype=[("id", "<u8"), ("code", "u1", (nsq,))])
            rec["id"] = ids
            rec["code"] = codes
            f.write(rec.tobytes())


def read_ref_results(path: str, nq: int, k: int):
    """Result file written by oracle/_ref/ref_tool (see ref_tool.cpp)."""
    rec = np.dtype([("count", "<u4"), ("lists", "<u4"), ("scanned", "<u8"),
                    ("nb", [("id", "<u8"), ("dist", "<f4")], (k,))])
    a = np.fromfile(path, dtype=rec, count=nq)
    return (a["nb"]["id"].copy(), a["nb"]["dist"].copy(), a["count"].copy(), a["scanned"].copy(),
            a["lists"].copy())


def ref_available() -> bool:
    return os.path.exists(REF_TOOL)


def ref_run(*args, timeout=3600) -> subprocess.CompletedProcess:
    return subprocess.run([REF_TOOL, *map(str, args)], check=True, capture_output=True, text=True,
                          timeout=timeout)
