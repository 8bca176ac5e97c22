"""B200-native IVF-PQ retrieval hot path of PipeRAG (arXiv 2403.05676).

Hand-written sm_100a kernels behind a C ABI (include/prag_gpu.h,
libprag_gpu.so); this package is the Python mirror of the reference's
retriever API. See DESIGN.md.
"""
from ._lib import (ConfigError, CudaError, FormatError, NoDeviceError, OutOfMemoryError, PragGpuError,
                   LIB_PATH, SYMBOLS, lib)
from .ivfpq import (BatchResult, Comm, GpuChunkEmbedder, GpuIndex, RetrievalPerfModel, ScoredId, SearchParams, SearchResult,
                    calibrate_gpu, calibrate_retrieval, device_count, load_index, load_perf_model, merge_topk,
                    plan_shards, plan_shard_ranges, search, select_nprobe, store_perf_model, TrainedIndex, TrainParams,
                    train_index, brute_force_search, recall_at_k)

__all__ = [
    "ConfigError", "CudaError", "FormatError", "NoDeviceError", "OutOfMemoryError", "PragGpuError", "LIB_PATH",
    "SYMBOLS", "lib", "BatchResult", "Comm", "GpuChunkEmbedder", "GpuIndex", "RetrievalPerfModel", "ScoredId", "SearchParams",
    "SearchResult", "calibrate_gpu", "calibrate_retrieval", "device_count", "load_index", "load_perf_model",
    "merge_topk", "plan_shards", "plan_shard_ranges", "search", "select_nprobe", "store_perf_model", "TrainedIndex", "TrainParams",
    "train_index", "brute_force_search", "recall_at_k",
]
