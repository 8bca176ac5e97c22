"""ctypes binding of libprag_gpu.so (the C ABI declared in include/prag_gpu.h).

The shared library is built in-tree by ``__graft_entry__.build()``
(``make -C paper_2403_05676_b200/csrc``). There is no fallback: importing the
package without the library raises, and every compute entry point fails with
``NoDeviceError`` on a host without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PRAG_GPU_LIB") or os.path.join(HERE, "libprag_gpu.so")  # override: A/B builds in tools/

OK, CONFIG, FORMAT, CUDA, NCCL, OOM, NO_DEVICE = range(7)


class PragGpuError(RuntimeError):
    code = -1


class ConfigError(PragGpuError):
    """Mirrors prag::ConfigError (common.hpp:23-25)."""
    code = CONFIG


class FormatError(PragGpuError):
    """Mirrors prag::FormatError (common.hpp:27-29)."""
    code = FORMAT


class CudaError(PragGpuError):
    code = CUDA


class OutOfMemoryError(PragGpuError):
    code = OOM


class NoDeviceError(PragGpuError):
    code = NO_DEVICE


_ERR = {CONFIG: ConfigError, FORMAT: FormatError, CUDA: CudaError, OOM: OutOfMemoryError,
        NO_DEVICE: NoDeviceError}


class IndexDesc(C.Structure):
    _fields_ = [("nlist", C.c_uint32), ("d", C.c_uint32), ("nsq", C.c_uint32), ("sub_dim", C.c_uint32),
                ("ntotal", C.c_uint64), ("ntotal_global", C.c_uint64), ("max_list_len", C.c_uint32),
                ("device", C.c_int32), ("shard_rank", C.c_int32), ("shard_world", C.c_int32),
                ("device_bytes", C.c_uint64), ("code_layout", C.c_uint32), ("reserved", C.c_uint32)]


class PerfModelC(C.Structure):
    _fields_ = [("slope_s", C.c_double), ("intercept_s", C.c_double), ("fit_residual_s", C.c_double),
                ("clamped", C.c_int32), ("reserved", C.c_int32)]


class Timings(C.Structure):
    _fields_ = [("coarse_ms", C.c_float), ("select_ms", C.c_float), ("plan_ms", C.c_float),
                ("scan_ms", C.c_float), ("final_ms", C.c_float), ("total_ms", C.c_float),
                ("scanned_bytes", C.c_uint64), ("work_items", C.c_uint64), ("coarse_window", C.c_uint64)]


class TrainParamsC(C.Structure):
    _fields_ = [("nlist", C.c_uint32), ("n_subquantizers", C.c_uint32), ("seed", C.c_uint64),
                ("kmeans_iterations", C.c_int32), ("reserved", C.c_int32), ("train_sample_cap", C.c_uint64)]


MEASURE_FN = C.CFUNCTYPE(C.c_double, C.c_uint32, C.c_void_p)

# (name, restype, argtypes) for every symbol include/prag_gpu.h declares.
P = C.c_void_p
SYMBOLS = [
    ("prag_gpu_last_error", C.c_char_p, []),
    ("prag_gpu_version", C.c_int, []),
    ("prag_gpu_device_count", C.c_int, []),
    ("prag_gpu_index_load", C.c_int, [C.c_char_p, C.c_int, C.POINTER(P)]),
    ("prag_gpu_index_load_shard", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(P)]),
    ("prag_gpu_index_from_host", C.c_int,
     [C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, P, C.c_int, C.POINTER(P)]),
    ("prag_gpu_index_synthetic", C.c_int,
     [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_double, P, P, C.c_int, C.POINTER(P)]),
    ("prag_gpu_train_index", C.c_int,
     [P, C.c_uint64, C.c_uint32, C.POINTER(TrainParamsC), C.c_int, P, P, P, P, P]),
    ("prag_gpu_index_store", C.c_int, [P, C.c_char_p]),
    ("prag_gpu_index_free", None, [P]),
    ("prag_gpu_index_describe", C.c_int, [P, C.POINTER(IndexDesc)]),
    ("prag_gpu_index_nlist", C.c_uint32, [P]),
    ("prag_gpu_index_list_sizes", C.c_int, [P, P]),
    ("prag_gpu_search", C.c_int, [P, P, C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, P]),
    ("prag_gpu_probe", C.c_int, [P, P, C.c_uint32, C.c_uint32, P, P, P]),
    ("prag_gpu_index_set_embeddings", C.c_int, [P, P, C.c_uint64]),
    ("prag_gpu_plan_create", C.c_int, [P, P, C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, P, C.POINTER(P)]),
    ("prag_gpu_plan_launch", C.c_int, [P, P]),
    ("prag_gpu_plan_free", None, [P]),
    ("prag_gpu_search_device", C.c_int, [P, P, C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, P]),
    ("prag_gpu_search_rerank", C.c_int, [P, P, C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, P]),
    ("prag_gpu_brute_force", C.c_int, [P, C.c_uint64, C.c_uint32, P, C.c_uint32, C.c_uint32, C.c_int, P, P, P]),
    ("prag_gpu_plan_shards", C.c_int, [P, C.c_uint32, C.c_uint32, P]),
    ("prag_gpu_plan_shard_ranges", C.c_int, [P, C.c_uint32, C.c_uint32, C.c_uint32, P, P]),
    ("prag_gpu_merge_topk", C.c_int,
     [P, P, P, P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, C.c_int, P]),
    ("prag_gpu_calibrate_retrieval", C.c_int,
     [P, P, C.c_uint32, C.c_uint32, P, C.c_uint32, C.c_int, C.c_int, C.POINTER(PerfModelC), P]),
    ("prag_gpu_calibrate_with", C.c_int,
     [MEASURE_FN, P, P, C.c_uint32, C.c_int, C.c_int, C.POINTER(PerfModelC)]),
    ("prag_gpu_select_nprobe", C.c_uint32, [C.POINTER(PerfModelC), C.c_double, C.c_uint32, C.c_double]),
    ("prag_gpu_set_scan_path", C.c_int, [P, C.c_int]),
    ("prag_gpu_set_sm_budget", C.c_int, [P, C.c_int]),
    ("prag_gpu_set_coarse_path", C.c_int, [P, C.c_int]),
    ("prag_gpu_set_profiling", C.c_int, [P, C.c_int]),
    ("prag_gpu_last_timings", C.c_int, [P, C.POINTER(Timings)]),
    ("prag_gpu_synthetic_decode", C.c_int, [P, C.c_uint64, C.c_uint32, P, P, P, C.c_uint64, P]),
    ("prag_gpu_synthetic_decode_sms", C.c_int, [P, C.c_uint64, C.c_uint32, P, P, P, C.c_uint64, C.c_uint32, P]),
    ("prag_gpu_embedder_create", C.c_int, [C.c_uint32, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(P)]),
    ("prag_gpu_embedder_free", None, [P]),
    ("prag_gpu_embed", C.c_int, [P, P, C.c_uint32, C.c_uint32, P, P]),
    ("prag_gpu_index_load_sharded", C.c_int, [C.c_char_p, P, C.c_int, C.POINTER(P)]),
    ("prag_gpu_index_group", C.c_int, [P, C.c_int, C.POINTER(P)]),
    ("prag_gpu_index_from_host_sharded", C.c_int,
     [C.c_uint32, C.c_uint32, C.c_uint32, P, P, P, P, P, P, C.c_int, C.POINTER(P)]),
    ("prag_gpu_index_synthetic_shard", C.c_int,
     [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_double, P, P, C.c_int, C.c_int, C.c_int,
      C.POINTER(P)]),
    ("prag_gpu_comm_unique_id", C.c_int, [P]),
    ("prag_gpu_comm_init", C.c_int, [P, C.c_int, C.c_int, C.c_int, C.POINTER(P)]),
    ("prag_gpu_comm_free", None, [P]),
    ("prag_gpu_index_attach_comm", C.c_int, [P, P]),
]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the search path)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SYMBOLS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().prag_gpu_last_error().decode(errors="replace")
        raise _ERR.get(rc, PragGpuError)(msg)
