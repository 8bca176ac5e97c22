/*
 * prag_gpu.h -- C ABI of the B200-native IVF-PQ retrieval hot path.
 *
 * Drop-in boundary for PipeRAG's retriever path. The reference has no FFI:
 * its extension point is the abstract C++ class prag::Retriever
 * (/root/reference/proj/include/prag/pipeline.hpp:200-208) wrapping the free
 * function prag::search (annindex.hpp:262-315) and the performance model
 * (perfmodel.hpp:92-157). Each entry point below names the reference
 * interface it replaces; include/prag_gpu.hpp wraps them back into the
 * reference's C++ shapes (SearchResult, Retriever) and INTEGRATION.md shows
 * the binding a maintainer adds.
 *
 * Around the search path, also bit-exact with the reference:
 * exact rerank (prag_gpu_search_rerank), brute force (prag_gpu_brute_force),
 * the index build (prag_gpu_train_index = prag::train_index), query
 * embedding (prag_gpu_embed = ChunkEmbedder::embed), the perf-model
 * calibration, and the synthetic decode step of the PipeRAG loop. The
 * PRAGRPC1 service lives in include/prag_gpu_service.hpp (C++ over this ABI).
 *
 * Conventions
 *  - Every function returns int status: 0 OK, 1 CONFIG (reference ConfigError),
 *    2 FORMAT (reference FormatError), 3 CUDA, 4 NCCL, 5 OOM, 6 NO_DEVICE.
 *    prag_gpu_last_error() returns the thread-local message of the last
 *    failure, worded like the reference's exception text.
 *  - Plain pointers and sizes only. Query/result pointers may be host or
 *    device memory (detected per pointer). With any host output the call
 *    returns only after results are in host memory; with all-device outputs
 *    the call is asynchronous on `stream` (a cudaStream_t, NULL = legacy).
 *  - The index is immutable after load; concurrent prag_gpu_search calls on
 *    different streams are safe (per-call workspaces from a pool).
 *  - There is no CPU fallback: without a CUDA device every compute entry
 *    point fails with status 6.
 */
#ifndef PRAG_GPU_H
#define PRAG_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PRAG_GPU_OK = 0,
    PRAG_GPU_CONFIG = 1,
    PRAG_GPU_FORMAT = 2,
    PRAG_GPU_CUDA = 3,
    PRAG_GPU_NCCL = 4,
    PRAG_GPU_OOM = 5,
    PRAG_GPU_NO_DEVICE = 6
};

typedef struct prag_gpu_index prag_gpu_index;

/* Shape and placement of a loaded index (or one shard of it). */
typedef struct prag_gpu_index_desc {
    uint32_t nlist;           /* IvfIndex::nlist (annindex.hpp:22)                 */
    uint32_t d;               /* IvfIndex::d                                       */
    uint32_t nsq;             /* PqCodebook::n_subquantizers (m, bytes per code)    */
    uint32_t sub_dim;         /* PqCodebook::sub_dim                               */
    uint64_t ntotal;          /* entries resident on this device                   */
    uint64_t ntotal_global;   /* entries in the whole index file                   */
    uint32_t max_list_len;    /* longest resident list                             */
    int32_t device;           /* CUDA ordinal                                      */
    int32_t shard_rank;       /* 0 when unsharded                                  */
    int32_t shard_world;      /* 1 when unsharded                                  */
    uint64_t device_bytes;    /* HBM held by the index                             */
    uint32_t code_layout;     /* 0 = plain [entry][m]; 1 = lane-skewed tiles (m=32,64) */
    uint32_t reserved;
} prag_gpu_index_desc;

/* Fitted retrieval-latency line; same fields and meaning as
 * prag::RetrievalPerfModel (perfmodel.hpp:19-26). */
typedef struct prag_gpu_perf_model {
    double slope_s;
    double intercept_s;
    double fit_residual_s;
    int32_t clamped;
    int32_t reserved;
} prag_gpu_perf_model;

/* Per-phase device time of the most recent search on an index with
 * profiling enabled (CUDA events on the search stream), milliseconds. */
typedef struct prag_gpu_timings {
    float coarse_ms;   /* K1: queries x centroids (tcgen05 GEMM or exact SIMT) */
    float select_ms;   /* K1b: per-query top-nprobe (window rescoring / select) */
    float plan_ms;     /* work-item plan (list sizes, prefix sums)          */
    float scan_ms;     /* K2+K3+K4: fused LUT build + list scan + top-k      */
    float final_ms;    /* per-query merge of partial top-k                  */
    float total_ms;    /* first event to last event                         */
    uint64_t scanned_bytes; /* algorithmic code bytes: sum scanned_vectors * m */
    uint64_t work_items;
    uint64_t coarse_window; /* lists rescored exactly by K1b (tensor-core path), summed over queries */
} prag_gpu_timings;

/* ---------------------------------------------------------------- errors */
const char* prag_gpu_last_error(void);
int prag_gpu_version(void);
/* Number of visible CUDA devices (0 on a host without a GPU; never fails). */
int prag_gpu_device_count(void);

/* ---------------------------------------------------------------- index */
/* Replaces prag::load_index (annindex.hpp:361-411): reads a PRAGIX01 file
 * and builds the HBM-resident list-major layout on `device`. Errors carry the
 * reference's FormatError wording and byte offsets. */
int prag_gpu_index_load(const char* pragix01_path, int device, prag_gpu_index** out);

/* Sharded load: keeps only the inverted lists that prag_gpu_plan_shards
 * assigns to `rank` of `world`; centroids and codebook are replicated so
 * every shard computes the identical probe set. */
int prag_gpu_index_load_shard(const char* pragix01_path, int device, int rank, int world,
                              prag_gpu_index** out);

/* Builds an index from host arrays in the reference's logical layout:
 * centroids[nlist][d], codewords[nsq][256][d/nsq], list_off[nlist+1] (entry
 * offsets into ids/codes), ids[ntotal], codes[ntotal][nsq]
 * (IvfIndex/PqCodebook, annindex.hpp:16-33, flattened). */
int prag_gpu_index_from_host(uint32_t nlist, uint32_t d, uint32_t nsq, const float* centroids,
                             const float* codewords, const uint64_t* list_off, const uint64_t* ids,
                             const uint8_t* codes, int device, prag_gpu_index** out);

/* Config-D fixture (BASELINE.json configs[3]): an index of `ntotal` entries
 * built directly in HBM, for the m = 32 / 64 fast path (k <= 32). List sizes
 * follow a log-normal skew (sigma) from SplitMix64(seed); entry g (global,
 * list-major) has chunk id g and code byte b = (W_{b/8} >> 8(b%8)) & 0xff with
 * W_i = splitmix64_finalize(seed + 8g + i + 0x9e3779b97f4a7c15). Centroids
 * [nlist][d] and codewords [nsq][256][d/nsq] are the caller's. No host copy
 * of the codes is ever made (1B entries = 64 GB at m = 64). */
int prag_gpu_index_synthetic(uint32_t nlist, uint32_t d, uint32_t nsq, uint64_t ntotal, uint64_t seed, double sigma,
                             const float* centroids, const float* codewords, int device, prag_gpu_index** out);

/* ---------------------------------------------------------------- build */
/* prag::TrainParams (annindex.hpp:152-160); reference defaults:
 * {nlist 64, n_subquantizers 0 (-> d/4), seed 7, kmeans_iterations 25,
 *  train_sample_cap 32768}. */
typedef struct prag_gpu_train_params {
    uint32_t nlist;
    uint32_t n_subquantizers;
    uint64_t seed;
    int32_t kmeans_iterations;
    int32_t reserved;
    uint64_t train_sample_cap;
} prag_gpu_train_params;

/* Replaces prag::train_index (annindex.hpp:164-241) on the device, bit-exact:
 * the same sample, k-means++ seeds, Lloyd iterations, IVF assignment, PQ
 * codebooks and codes as the reference's scalar code. vectors: n x d fp32
 * row-major (host or device). Outputs (host or device, each independently) in
 * the flattened IvfIndex/PqCodebook layout prag_gpu_index_from_host takes:
 * centroids[nlist][d], codewords[nsq][256][d/nsq] (unused tail codes zero),
 * list_off[nlist+1], ids[n] and codes[n][nsq] list-major, each list in vector
 * order (ids are vector indices). Errors: the reference's ConfigError texts;
 * n must be < 2^32. */
int prag_gpu_train_index(const float* vectors, uint64_t n, uint32_t d, const prag_gpu_train_params* params,
                         int device, float* centroids, float* codewords, uint64_t* list_off, uint64_t* ids,
                         uint8_t* codes);

/* Replaces prag::store_index (annindex.hpp:335-359): writes the resident
 * index as PRAGIX01 (byte-identical to the file it was loaded from, or to
 * store_index of the same IvfIndex/PqCodebook). Full (unsharded) indexes with
 * the plain code layout only. */
int prag_gpu_index_store(const prag_gpu_index* index, const char* pragix01_path);

void prag_gpu_index_free(prag_gpu_index* index);
int prag_gpu_index_describe(const prag_gpu_index* index, prag_gpu_index_desc* out);
/* IvfIndex::nlist, as prag::Retriever::nlist() (pipeline.hpp:207). */
uint32_t prag_gpu_index_nlist(const prag_gpu_index* index);
/* Resident list lengths (host array of nlist). */
int prag_gpu_index_list_sizes(const prag_gpu_index* index, uint64_t* out_sizes);

/* ---------------------------------------------------------------- search */
/* Replaces prag::search(index, codebook, query, {nprobe, k, false})
 * (annindex.hpp:262-315) for a batch of nq queries (row-major nq x d).
 * Validation as annindex.hpp:265-268: k >= 1 and 1 <= nprobe <= nlist, else
 * CONFIG. Outputs per query q: out_ids[q*k + i], out_dist[q*k + i] for
 * i < out_count[q] = min(k, candidates), ascending (distance, chunk_id);
 * out_scanned_vectors[q] = SearchResult::scanned_vectors (may be NULL).
 * SearchResult::scanned_lists is always nprobe (annindex.hpp:284). */
int prag_gpu_search(prag_gpu_index* index, const float* queries, uint32_t nq, uint32_t nprobe,
                    uint32_t k, uint64_t* out_ids, float* out_dist, uint32_t* out_count,
                    uint64_t* out_scanned_vectors, void* stream);

/* prag_gpu_search for callers whose queries and outputs are all device
 * memory (asynchronous on `stream`): the same work without the per-call
 * pointer-kind queries. Passing host memory here is undefined. */
int prag_gpu_search_device(prag_gpu_index* index, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t k,
                           uint64_t* out_ids, float* out_dist, uint32_t* out_count, uint64_t* out_scanned,
                           void* stream);

/* A captured search (CUDA graph) for a fixed batch shape and fixed device
 * buffers: create once with the buffers a serving loop reuses, then
 * prag_gpu_plan_launch per batch after writing the queries into them. One
 * graph launch replaces the five kernel launches (host cost), results are
 * identical to prag_gpu_search. The batch must fit one pass. */
typedef struct prag_gpu_plan prag_gpu_plan;
int prag_gpu_plan_create(prag_gpu_index* index, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t k,
                         uint64_t* out_ids, float* out_dist, uint32_t* out_count, uint64_t* out_scanned,
                         void* stream, prag_gpu_plan** out);
int prag_gpu_plan_launch(prag_gpu_plan* plan, void* stream);
void prag_gpu_plan_free(prag_gpu_plan* plan);

/* Exact rerank (SearchParams::exact_rerank, annindex.hpp:307-312): raw
 * embeddings [n][d] fp32 row-major indexed by chunk id (host or device
 * pointer; copied into HBM). Every resident chunk id must be < n. n = 0
 * detaches. */
int prag_gpu_index_set_embeddings(prag_gpu_index* index, const float* embeddings, uint64_t n);
/* prag::search(..., {nprobe, k, true}, &embeddings): the probed candidates'
 * distances replaced by the full-precision squared_l2(embeddings[id], query)
 * before the (distance, chunk_id) top-k. Same arguments and outputs as
 * prag_gpu_search; PRAG_GPU_CONFIG "search: exact_rerank requires raw
 * embeddings" when none are attached. */
int prag_gpu_search_rerank(prag_gpu_index* index, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t k,
                           uint64_t* out_ids, float* out_dist, uint32_t* out_count, uint64_t* out_scanned,
                           void* stream);

/* prag::brute_force_search (annindex.hpp:244-257) on the device: exact
 * top-k of n rows [n][d] (host or device) by full-precision squared L2 in the
 * reference's rounding, ties by lower row id; outputs [nq][k] host or device.
 * For recall evaluation (acceptance C1/C2), not the serving path. */
int prag_gpu_brute_force(const float* vectors, uint64_t n, uint32_t d, const float* queries, uint32_t nq,
                         uint32_t k, int device, uint64_t* out_ids, float* out_dist, uint32_t* out_count);

/* Coarse quantizer only (annindex.hpp:277-281): the first nprobe lists of
 * each query in (distance, list id) order, out_lists[q*nprobe + p]. */
int prag_gpu_probe(prag_gpu_index* index, const float* queries, uint32_t nq, uint32_t nprobe,
                   uint32_t* out_lists, float* out_dist, void* stream);

/* ------------------------------------------------------ multi-GPU pieces */
/* Placement of lists on `world` shards by bytes (|l| * m). Large lists (at
 * least 4x the mean list size and 1024 entries per stripe) are STRIPED over
 * all ranks -- rank r holds entries [len*r/world, len*(r+1)/world) -- and get
 * out_owner = world; the rest go whole by LPT: descending size (ties by lower
 * id), each to the least-loaded shard (ties by lower rank), the striped
 * loads counted first. Host-only; never touches a GPU. */
int prag_gpu_plan_shards(const uint64_t* list_sizes, uint32_t nlist, uint32_t world,
                         uint32_t* out_owner);
/* The same placement as the entry range [out_begin[l], out_end[l]) of every
 * list held by `rank` (empty when the list is not resident there): what
 * load_shard / synthetic_shard / the sharded loaders keep. */
int prag_gpu_plan_shard_ranges(const uint64_t* list_sizes, uint32_t nlist, uint32_t world, uint32_t rank,
                               uint64_t* out_begin, uint64_t* out_end);

/* Exact top-k of the union of `nparts` per-shard top-k lists, per query.
 * Inputs device or host: ids/dist [nparts][nq][kin], count [nparts][nq];
 * scanned [nparts][nq] summed into out_scanned (both may be NULL). */
int prag_gpu_merge_topk(const uint64_t* ids, const float* dist, const uint32_t* count,
                        const uint64_t* scanned, uint32_t nparts, uint32_t nq, uint32_t kin,
                        uint32_t k, uint64_t* out_ids, float* out_dist, uint32_t* out_count,
                        uint64_t* out_scanned, int device, void* stream);

/* ----------------------------------------- list-sharded search (8e) */
/* The reference's Retriever is called by C++ (pipeline.hpp:221-238, :496;
 * service.hpp:338), so the multi-GPU path is behind this ABI too, in two
 * forms (lists placed by LPT on bytes, centroids and codebook
 * replicated, per-shard K1-K4, one exchange of the per-shard top-k, exact
 * merge by (distance, chunk id) -- bit-identical to the unsharded search):
 *
 * (1) One process driving several GPUs: a GROUP handle. prag_gpu_search /
 *     _device / _rerank / plan_* / calibrate on it run every shard on its
 *     own device and stream, then ONE kernel on the root device (devices[0])
 *     reads each shard's top-k over NVLink peer memory and merges them (the
 *     gather fused into the merge; shards without peer access are copied to
 *     the root first). A group is a prag_gpu_index everywhere in this ABI
 *     (GpuRetriever, the service, the perf model take it unchanged). Devices
 *     may repeat (several shards on one GPU). */
int prag_gpu_index_load_sharded(const char* pragix01_path, const int* devices, int n_devices,
                                prag_gpu_index** out);
/* The same from host arrays in prag_gpu_index_from_host's layout. */
int prag_gpu_index_from_host_sharded(uint32_t nlist, uint32_t d, uint32_t nsq, const float* centroids,
                                     const float* codewords, const uint64_t* list_off, const uint64_t* ids,
                                     const uint8_t* codes, const int* devices, int n_devices,
                                     prag_gpu_index** out);
/* Group of already-built shards (load_shard / synthetic_shard ranks 0..n-1
 * of world n, any devices); takes ownership of the shard handles. */
int prag_gpu_index_group(prag_gpu_index* const* shards, int n, prag_gpu_index** out);

/* Rank `rank` of `world` of the synthetic index prag_gpu_index_synthetic
 * builds from the same arguments (lists placed by prag_gpu_plan_shards on the
 * synthetic list sizes; every entry keeps its global chunk id and code). */
int prag_gpu_index_synthetic_shard(uint32_t nlist, uint32_t d, uint32_t nsq, uint64_t ntotal, uint64_t seed,
                                   double sigma, const float* centroids, const float* codewords, int rank,
                                   int world, int device, prag_gpu_index** out);

/* (2) One process per GPU (torchrun / MPI ranks): an NCCL communicator
 *     (NCCL is resolved at run time: libnccl.so.2, the copy the process
 *     already has loaded if any). Attach it to the rank's shard; from then on
 *     prag_gpu_search / plans on that shard are COLLECTIVE: every rank passes
 *     the same queries, runs K1-K4 on its lists, the per-shard top-k blocks are
 *     exchanged with one ncclAllGather on the search stream, and every rank
 *     gets the merged global result. Graph-capturable (prag_gpu_plan_create,
 *     called by all ranks). */
typedef struct prag_gpu_comm prag_gpu_comm;
int prag_gpu_comm_unique_id(uint8_t out_id[128]);   /* ncclGetUniqueId, on one rank */
int prag_gpu_comm_init(const uint8_t id[128], int world, int rank, int device, prag_gpu_comm** out);
void prag_gpu_comm_free(prag_gpu_comm* comm);
/* shard: rank r of world w (load_shard / synthetic_shard) with comm rank r of
 * w on the same device; comm NULL detaches. The comm must outlive its use. */
int prag_gpu_index_attach_comm(prag_gpu_index* shard, prag_gpu_comm* comm);

/* ------------------------------------------------- performance model */
/* Replaces prag::calibrate_retrieval (perfmodel.hpp:92-117) fed with the GPU
 * latency curve: for each nprobe in grid (sorted, deduplicated; >= 2 values,
 * repeats >= 3), `warmups` untimed then `repeats` timed batch searches of the
 * nq host queries; the median batch latency in seconds per point is fitted
 * with least squares; negative coefficients are clamped to 0.
 * If out_latency_s is non-NULL it receives the medians (one per unique
 * grid value, ascending). */
int prag_gpu_calibrate_retrieval(prag_gpu_index* index, const float* queries, uint32_t nq,
                                 uint32_t k, const uint32_t* nprobe_grid, uint32_t grid_len,
                                 int repeats, int warmups, prag_gpu_perf_model* out_model,
                                 double* out_latency_s);

/* Same fit over caller-supplied timings: `measure(nprobe, ctx)` returns
 * seconds (the std::function hook of perfmodel.hpp:92). */
typedef double (*prag_gpu_measure_fn)(uint32_t nprobe, void* ctx);
int prag_gpu_calibrate_with(prag_gpu_measure_fn measure, void* ctx, const uint32_t* nprobe_grid,
                            uint32_t grid_len, int repeats, int warmups,
                            prag_gpu_perf_model* out_model);

/* prag::select_nprobe (perfmodel.hpp:148-157). */
uint32_t prag_gpu_select_nprobe(const prag_gpu_perf_model* model, double budget_s, uint32_t nlist,
                                double safety_margin);

/* ------------------------------------------------------------ profiling */
/* Scan-path selection: 0 = automatic (lane-skewed fused fast path for
 * m = 32 / 64 and k <= 32, generic otherwise), 1 = always the generic path
 * (used by the parity suite to check both paths against each other). */
/* SM budget of the persistent search kernels (the list scan's grid, the
 * batch-1 kernel): searches size their grids to min(sms, device SMs) so
 * they run beside work pinned to the other SMs (config E). 0 = every SM. */
int prag_gpu_set_sm_budget(prag_gpu_index* index, int sms);
int prag_gpu_set_scan_path(prag_gpu_index* index, int path);
/* Coarse-quantizer selection: 0 = automatic (tcgen05 tensor-core pre-filter
 * + exact rescoring of the boundary window when nlist % 128 == 0,
 * d % 32 == 0 and nprobe <= 256), 1 = always the exact SIMT scan of every
 * centroid. Both return identical probe lists. */
int prag_gpu_set_coarse_path(prag_gpu_index* index, int path);
int prag_gpu_set_profiling(prag_gpu_index* index, int enabled);
int prag_gpu_last_timings(const prag_gpu_index* index, prag_gpu_timings* out);

/* ------------------------------------------------ query embedding */
/* Device-resident prag::ChunkEmbedder (tokendb.hpp:84-124), the step before
 * search in LocalRetriever::retrieve (pipeline.hpp:227). Token unit vectors
 * for ids [0, vocab) are computed on the host exactly as token_unit_vector
 * (tokendb.hpp:63-80) and kept in HBM; prag_gpu_embed reproduces embed()
 * bit for bit (double accumulation in token order, sequential squared norm,
 * IEEE sqrt/div, fp32 rounding; e_0 for an all-PAD chunk). */
typedef struct prag_gpu_embedder prag_gpu_embedder;
int prag_gpu_embedder_create(uint32_t d, uint64_t seed, uint32_t vocab, int device, prag_gpu_embedder** out);
void prag_gpu_embedder_free(prag_gpu_embedder* embedder);
/* tokens: nchunks x m token ids (PAD = 0 skipped), host or device; out:
 * nchunks x d floats, host or device. With host tokens any id is accepted:
 * ids >= vocab get their vectors computed on the host for that call, as
 * ChunkEmbedder::embed does for every id. Device tokens must be < vocab
 * (CONFIG otherwise, reported when any pointer is host memory). */
int prag_gpu_embed(prag_gpu_embedder* embedder, const uint32_t* tokens, uint32_t nchunks, uint32_t m, float* out,
                   void* stream);

/* ------------------------------------------------- config-E harness */
/* One synthetic decode step on `stream` (device pointers): y[r] = W[r] . x
 * for a rows x cols fp32 weight matrix, plus a streaming read of kv_floats
 * of KV cache. The memory-bound stand-in for a RETRO decode step that the
 * PipeRAG pipeline overlaps retrieval with; it replaces the reference's
 * SyntheticGenerator (generator.hpp:220-252), whose per-token cost is affine
 * in position. Not part of the retrieval path. y must hold rows + 1 floats. */
int prag_gpu_synthetic_decode(const float* weights, uint64_t rows, uint32_t cols, const float* x, float* y,
                              const float* kv, uint64_t kv_floats, void* stream);
/* The same decode step on exactly `sms` SMs (one 1024-thread CTA per SM),
 * leaving the other SMs free for retrieval on a side stream (config E). */
int prag_gpu_synthetic_decode_sms(const float* weights, uint64_t rows, uint32_t cols, const float* x, float* y,
                                  const float* kv, uint64_t kv_floats, uint32_t sms, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PRAG_GPU_H */
