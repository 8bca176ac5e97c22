// internal.h -- shared declarations of the prag_gpu library (not public ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "prag_gpu.h"

namespace pg {

// ------------------------------------------------- programmatic launches
// The search kernels form one dependent chain on a stream. Launched with
// programmatic stream serialization, kernel N+1 is scheduled while kernel N
// drains; it runs its index-only prologue, then pdl_wait() before touching
// kernel N's outputs. pdl_trigger() marks where a kernel lets its dependent
// launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Chain trace (debug build only: make EXTRA=-DPRAG_CHAIN_TRACE). Per kernel
// of the search chain, per CTA (< kChainCtas) and warp: the CTA's start, the
// warp's PDL-wait return and the warp's end, as globaltimer values in plain
// stores (no atomics: the trace must not serialise the kernels it times);
// tools/chain_trace.py reads them back with prag_gpu_debug_chain_trace. Ids:
// 0 K1, 1 K1b, 2 K2, 3 planner CTA, 4 K3, 5 K4; 6.. phase marks inside a
// kernel (CT_MARK: the time a warp passed the mark, in the "waited" field).
#ifdef PRAG_CHAIN_TRACE
constexpr int kChainKernels = 20;
constexpr uint32_t kChainCtas = 8192, kChainWarps = 32;
constexpr size_t kChainWords = size_t(kChainKernels) * kChainCtas * kChainWarps * 3;
static __constant__ unsigned long long* c_chain;
__device__ __forceinline__ unsigned long long ct_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long* ct_slot(int k) {
    const uint32_t cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (cta >= kChainCtas || (threadIdx.x & 31u) != 0) return nullptr;
    return c_chain + ((size_t(k) * kChainCtas + cta) * kChainWarps + (threadIdx.x >> 5)) * 3;
}
#define CT_BEGIN const unsigned long long ct_t0 = ::pg::ct_now()
#define CT_WAITED(k)                                          \
    do {                                                      \
        unsigned long long* p_ = ::pg::ct_slot(k);            \
        if (p_) {                                             \
            p_[0] = ct_t0;                                    \
            p_[1] = ::pg::ct_now();                           \
        }                                                     \
    } while (0)
#define CT_MARK(k) CT_WAITED(k)
#define CT_END(k)                                             \
    do {                                                      \
        unsigned long long* p_ = ::pg::ct_slot(k);            \
        if (p_) p_[2] = ::pg::ct_now();                       \
    } while (0)
#define CT_BIND_FN(name) \
    void name(void* p) { cudaMemcpyToSymbol(c_chain, &p, sizeof(p)); }
void ct_bind_coarse(void* p);
void ct_bind_skew(void* p);
void ct_bind_kernels(void* p);
#else
#define CT_BEGIN
#define CT_MARK(k)
#define CT_WAITED(k)
#define CT_END(k)
#endif

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
// and size: a hot-path launch does not pay the driver call every time.
cudaError_t ensure_smem(const void* kernel, size_t bytes);

struct Status {
    int code = PRAG_GPU_OK;
    static Status ok() { return {}; }
};

#define PG_CUDA(expr)                                                                      \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess) {                                                           \
            ::pg::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " + \
                            __FILE__ + ":" + std::to_string(__LINE__) + " (" #expr ")");  \
            return _e == cudaErrorMemoryAllocation ? PRAG_GPU_OOM : PRAG_GPU_CUDA;         \
        }                                                                                  \
    } while (0)

// Every extern "C" int entry point runs inside PG_API_BEGIN / PG_API_END:
// no C++ exception (a host allocation sized from a corrupt header, a
// std::vector growth) crosses the C ABI; it becomes a status code instead.
#define PG_API_BEGIN try {
#define PG_API_END                                                              \
    }                                                                           \
    catch (const std::bad_alloc&) {                                             \
        ::pg::set_error("out of host memory");                                  \
        return PRAG_GPU_OOM;                                                    \
    }                                                                           \
    catch (const std::length_error& e) {                                        \
        ::pg::set_error(std::string("allocation too large: ") + e.what());      \
        return PRAG_GPU_OOM;                                                    \
    }                                                                           \
    catch (const std::exception& e) {                                           \
        ::pg::set_error(std::string("internal error: ") + e.what());            \
        return PRAG_GPU_CONFIG;                                                 \
    }                                                                           \
    catch (...) {                                                               \
        ::pg::set_error("internal error: unknown exception");                   \
        return PRAG_GPU_CONFIG;                                                 \
    }

#define PG_TRY(expr)                      \
    do {                                  \
        int _rc = (expr);                 \
        if (_rc != PRAG_GPU_OK) return _rc; \
    } while (0)

// ------------------------------------------------------------- host index
// De-interleaved (SoA, list-major) image of a PRAGIX01 file
// (annindex.hpp:335-359 AoS -> arrays).
struct HostIndex {
    uint32_t nlist = 0, d = 0, nsq = 0, sub_dim = 0;
    std::vector<float> centroids;   // [nlist][d]
    std::vector<float> codewords;   // [nsq][256][sub_dim]
    std::vector<uint64_t> list_off; // [nlist+1]
    std::vector<uint64_t> ids;      // [ntotal]
    std::vector<uint8_t> codes;     // [ntotal][nsq]
    uint64_t ntotal_global = 0;
};

// Parses PRAGIX01 (annindex.hpp:361-411). keep = {begin[nlist], end[nlist]}
// selects each list's resident entry range (sharding; empty ranges are
// skipped on disk). Returns status, error text set.
struct KeepRanges {
    std::vector<uint64_t> begin, end;
};
int read_pragix01(const std::string& path, HostIndex& out, const KeepRanges* keep);
int read_pragix01_list_sizes(const std::string& path, std::vector<uint64_t>& sizes);
// Shard placement (index_io.cpp): owner[l] = the rank holding list l whole,
// or world when the list is striped over all ranks; plan_shard_ranges gives
// rank's entry range [begin, end) of every list (empty when not resident).
void plan_shards_lpt(const uint64_t* sizes, uint32_t nlist, uint32_t world, uint32_t* owner);
void plan_shard_ranges(const uint64_t* sizes, uint32_t nlist, uint32_t world, uint32_t rank, uint64_t* begin,
                       uint64_t* end);
inline uint64_t stripe_begin(uint64_t len, uint32_t world, uint32_t r) {
    return uint64_t((unsigned __int128)len * r / world);
}
inline uint64_t stripe_end(uint64_t len, uint32_t world, uint32_t r) { return stripe_begin(len, world, r + 1); }

// ----------------------------------------------------------- device index
constexpr uint32_t kListPad = 32;  // lists padded to a multiple of 32 entries

struct DeviceIndex {
    uint32_t nlist = 0, d = 0, nsq = 0, sub_dim = 0;
    uint64_t ntotal = 0;       // real resident entries
    uint64_t npadded = 0;      // padded slots
    uint32_t max_list_len = 0;
    float* centroids = nullptr;   // [nlist][d]
    float* centroidsT = nullptr;  // [d][nlist] (coalesced coarse scan)
    float* centroids4 = nullptr;  // [d/4][nlist][4] (vectorised coarse scan, d % 4 == 0)
    float* codewordsT = nullptr;  // [nsq][sub_dim][256]
    uint64_t* list_off = nullptr; // [nlist+1] padded slot offsets
    uint32_t* list_len = nullptr; // [nlist]
    uint64_t* ids = nullptr;      // [npadded]
    uint8_t* codes = nullptr;     // plain: [npadded][nsq]; skewed: see kernels.cu
    uint32_t code_layout = 0;     // 1: skew_codes present (m = 32 / 64 fast path)
    float* codewords = nullptr;   // [nsq][256][sub_dim] (LUT-image kernel)
    uint64_t* skew_off = nullptr; // [nlist+1] tile offsets into skew_codes
    uint8_t* skew_codes = nullptr;
    float* cent_tc = nullptr;     // K1 A operand: fp32 centroids in UMMA core-matrix order (split hi/lo in SMEM)
    float* cent_norm = nullptr;   // [nlist] ||c||^2
    bool tc_ok = false;           // tensor-core coarse quantizer usable for this shape
    bool plain_codes = true;      // codes[] present (generic path); false for device-built synthetic indexes
};

// ------------------------------------------------------------ workspace
struct Workspace {
    int device = 0;
    cudaEvent_t done = nullptr;   // recorded after the last kernel using it
    cudaStream_t last_stream = nullptr;
    bool busy = false;
    // device buffers (grown on demand)
    void* buf = nullptr;
    size_t buf_bytes = 0;
    void* stage = nullptr;        // query/output staging
    size_t stage_bytes = 0;
    // pinned host staging
    void* host = nullptr;
    size_t host_bytes = 0;
    // the last async H2D out of `host` (pageable queries staged through it):
    // the next write into `host` waits for it (a later chunk or call must not
    // overwrite queries a queued copy has not read yet)
    cudaEvent_t host_ev = nullptr;
    bool host_pending = false;
    // list sharding (shard.cu): the per-shard top-k block / gathered blocks,
    // and two events for cross-stream (cross-device) hand-offs
    void* xbuf = nullptr;
    size_t xbuf_bytes = 0;
    cudaEvent_t xev = nullptr, xev2 = nullptr;
    // batch-1 kernel (batch1.cu): grid-barrier and finish-ticket counters
    unsigned* sync = nullptr;
    // profiling events
    cudaEvent_t ev[8] = {};
    unsigned long long* win_stat = nullptr;  // profiling: sum of K1b window sizes
};

// A captured search over fixed device buffers, serving prag_gpu_search calls
// with host queries and outputs of one (nq, nprobe, k, stream) shape.
struct HostPlan {
    uint32_t nq = 0, nprobe = 0, k = 0;
    cudaStream_t stream = nullptr;
    prag_gpu_plan* plan = nullptr;
    float* dq = nullptr;         // [nq][d]
    char* dout = nullptr;        // ids | dist | count | scanned (Carver offsets)
    char* hout = nullptr;        // pinned copy of dout
    size_t out_bytes = 0;
    bool busy = false;
    uint64_t last_use = 0;
};

struct SearchPlanSizes {
    uint32_t nq_chunk;     // queries per pass
    uint64_t cand_cap;     // candidate slots per pass
    uint64_t item_cap;     // work items per pass
};

}  // namespace pg

struct prag_gpu_index {
    int device = 0;
    int shard_rank = 0, shard_world = 1;
    uint64_t ntotal_global = 0;
    pg::DeviceIndex dev;
    std::vector<uint64_t> host_list_len;          // resident sizes
    std::vector<uint64_t> top_prefix;             // prefix sums of sizes sorted desc
    uint64_t device_bytes = 0;
    bool profiling = false;
    int scan_path = 0;                            // 0 auto, 1 force generic
    int coarse_path = 0;                          // 0 auto (tensor cores when eligible), 1 force exact SIMT
    int sm_budget = 0;                            // persistent search grids: 0 = every SM
    prag_gpu_timings last{};
    float* emb = nullptr;                         // raw embeddings [emb_n][d] for exact rerank (annindex.hpp:307-312)
    uint64_t emb_n = 0;
    std::mutex mu;                                // guards pool and `last`
    std::vector<pg::Workspace*> pool;
    // prefix sums of the WHOLE index's list sizes sorted desc (== top_prefix
    // unless this is a shard): pass sizes that every rank agrees on
    std::vector<uint64_t> global_top_prefix;
    // --- list sharding (shard.cu)
    // group handle: a list-sharded index spanning these shards (owned; shard
    // r holds rank r of world shards.size(), possibly on different devices).
    // dev holds only the shape (no device arrays); `device` is the root.
    std::vector<prag_gpu_index*> shards;
    std::vector<cudaStream_t> shard_streams;      // one per shard, on its device
    std::vector<uint8_t> peer_direct;             // root's merge reads shard r's memory directly
    // multi-process: this shard is rank comm->rank of a distributed index;
    // prag_gpu_search on it is collective (NCCL all-gather + merge)
    prag_gpu_comm* comm = nullptr;
    // host-buffer searches replayed as captured plans (capi.cu host_plan_search)
    std::vector<pg::HostPlan*> host_plans;
    bool is_group() const { return !shards.empty(); }
};

namespace pg {

// kernels.cu launchers (all asynchronous on `s`)
struct SearchBuffers {
    // inputs
    const float* queries;   // device [nq][d]
    uint32_t nq, nprobe, k;
    // outputs (device)
    uint64_t* out_ids;
    float* out_dist;
    uint32_t* out_count;
    uint64_t* out_scanned;
    // scratch (device)
    float* coarse_dist;     // [nq][nlist]
    uint32_t* probe;        // [nq][nprobe]
    float* probe_dist;      // [nq][nprobe]
    uint64_t* q_cand_off;   // [nq+1]
    uint4* items;           // [item_cap]
    uint32_t* num_items;    // [1]
    uint32_t* item_cursor;  // [1]
    float* cand_dist;       // [cand_cap]
    uint32_t* cand_entry;   // [cand_cap]
    uint32_t* sort_scratch; // generic select scratch
    uint64_t item_cap, cand_cap;
};

int launch_coarse(const DeviceIndex& ix, const float* queries, uint32_t nq, float* out, cudaStream_t s);
int launch_select_probe(const DeviceIndex& ix, const float* coarse, uint32_t nq, uint32_t nprobe,
                        uint32_t* probe, float* probe_dist, uint32_t* gkey, uint64_t* gtie, cudaStream_t s);
int launch_plan(const DeviceIndex& ix, const SearchBuffers& b, cudaStream_t s);
int launch_scan(const DeviceIndex& ix, const SearchBuffers& b, cudaStream_t s, int grid, float* glut);
// exact rerank (annindex.hpp:307-312): every candidate's distance becomes
// squared_l2(emb[chunk_id], q) at full precision; max_cand_q bounds a query's candidates
int launch_rerank(const DeviceIndex& ix, const SearchBuffers& b, const float* emb, uint64_t max_cand_q,
                  cudaStream_t s);
// brute_force_search (annindex.hpp:244-257) for nq device queries over n device rows;
// dist is [nq][n] scratch, gkey/gtie [nq][pw] with pw = pow2 >= k
int max_chunk_id(const uint64_t* ids, uint64_t n, uint64_t* out);
int launch_brute_force(const float* emb, uint64_t n, uint32_t d, const float* queries, uint32_t nq, uint32_t k,
                       float* dist, uint32_t* gkey, uint64_t* gtie, uint32_t pw, uint64_t* out_ids, float* out_dist,
                       uint32_t* out_count, cudaStream_t s);
int launch_final(const DeviceIndex& ix, const SearchBuffers& b, uint32_t* gkey, uint64_t* gtie, uint32_t pw,
                 cudaStream_t s);
int launch_merge(const uint64_t* ids, const float* dist, const uint32_t* count, const uint64_t* scanned,
                 uint32_t nparts, uint32_t nq, uint32_t kin, uint32_t k, uint64_t* out_ids, float* out_dist,
                 uint32_t* out_count, uint64_t* out_scanned, uint32_t* ckey, uint64_t* ctie, uint32_t* gkey,
                 uint64_t* gtie, uint32_t pw, cudaStream_t s);
uint32_t scan_chunk();
// fast path (scan_skew.cu)
// K2 + planner: LUTs of every (query, probed list) pair, and (one extra CTA)
// the scan's work items, scanned_vectors and per-query threshold/pool reset
int launch_lut_images(const DeviceIndex& ix, const float* queries, const uint32_t* probe, uint32_t nq,
                      uint32_t nprobe, float* luts, uint32_t it_tiles, uint64_t* scanned, uint4* items,
                      uint32_t* num_items, uint32_t* cursor, uint32_t* q_item_off, uint32_t* gthr,
                      uint32_t* pair_off, uint64_t item_cap, uint32_t scan_grid, cudaStream_t s);
int launch_scan_skew(const DeviceIndex& ix, const uint4* items, const uint32_t* num_items, uint32_t* cursor,
                     const uint32_t* probe, const float* images, uint32_t nprobe, uint32_t k, uint32_t* gthr,
                     uint32_t* pool_key, uint64_t* pool_id, int grid, cudaStream_t s);
// K4: per query, exact top-k of its items' pool slots (k entries per item,
// [q_item_off[q] * k, q_item_off[q + 1] * k)); count = min(scanned[q], k)
int launch_select_pool(const uint32_t* pool_key, const uint64_t* pool_id, const uint64_t* ids, const uint64_t* scanned,
                       const uint32_t* q_item_off, const uint32_t* gthr, uint32_t nq, uint32_t k, uint64_t* out_ids,
                       float* out_dist, uint32_t* out_count, uint32_t* gkey, uint64_t* gtie, uint32_t pw,
                       cudaStream_t s);
uint32_t skew_item_tiles(uint64_t est_tiles, uint32_t grid);
uint32_t skew_min_item_tiles();
size_t skew_lut_bytes(uint32_t m);
uint32_t skew_warps(uint32_t m);
void build_skew_layout(const HostIndex& h, uint32_t m, std::vector<uint64_t>& skew_off, std::vector<uint8_t>& out);
uint32_t sort_cap();
// tensor-core coarse quantizer (coarse_tc.cu)
bool tc_coarse_supported(uint32_t nlist, uint32_t d);
float tc_bound_c(uint32_t d);
void build_tc_centroids(const float* cent, uint32_t nlist, uint32_t d, std::vector<float>& out,
                        std::vector<float>& norms);
uint32_t tc_slices(uint32_t d);
// K1 writes partial[tc_slices(d)][nq][nlist]; K1b consumes it (and uses slice 0 as scratch)
int launch_coarse_tc(const DeviceIndex& ix, const float* queries, uint32_t nq, float* partial, cudaStream_t s);
int launch_select_window(const DeviceIndex& ix, float* partial, const float* queries, uint32_t nq, uint32_t nprobe,
                         uint32_t* probe, float* probe_dist, unsigned long long* win_stat, cudaStream_t s);
constexpr uint32_t kTcMaxNprobe = 256;
// device-built synthetic index (synth_index.cu)
void synth_list_sizes(uint32_t nlist, uint64_t ntotal, uint64_t seed, double sigma, std::vector<uint64_t>& sizes);
// gbase[l]: global list-major position of list l's entry 0; rlen[l]: its
// resident length (0 for lists another shard holds)
int launch_synth_codes(uint32_t m, const uint64_t* gbase, const uint64_t* rlen, const uint64_t* skew_off, uint32_t nlist,
                       uint64_t seed, uint8_t* out, uint64_t ntiles, uint64_t* ids, const uint64_t* pad_off,
                       uint64_t npadded);
size_t select_smem_bytes();

}  // namespace pg

namespace pg {

// ------------------------------------------------- orchestration (capi.cu)
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

struct Carver {
    char* base;
    size_t off = 0;
    template <typename T>
    T* take(size_t n) {
        off = (off + 255) & ~size_t(255);
        T* p = reinterpret_cast<T*>(base + off);
        off += std::max<size_t>(n * sizeof(T), 16);
        return p;
    }
};

int sm_count(int device);
int search_sms(const prag_gpu_index* ix);
// batch-1 single-launch search (batch1.cu)
bool search1_eligible(const DeviceIndex& d, uint32_t nq, uint32_t nprobe, uint32_t k, int sms);
size_t search1_scratch_bytes(const DeviceIndex& d, uint32_t nprobe, int grid);
int launch_search1(const DeviceIndex& d, const float* dq, uint32_t nprobe, uint32_t k, uint64_t* o_ids,
                   float* o_dist, uint32_t* o_count, uint64_t* o_scanned, void* scratch, unsigned* sync, int grid,
                   cudaStream_t s);
int require_device(int device);
bool is_device_ptr(const void* p);
bool is_pinned_host(const void* p);
uint32_t pow2_at_least(uint64_t v);
void free_device_index(DeviceIndex& d);
int upload(prag_gpu_index* ix, const HostIndex& h);
int finish_load(std::unique_ptr<prag_gpu_index>& ix, HostIndex& h, int device, prag_gpu_index** out);
Workspace* acquire_ws(prag_gpu_index* ix, cudaStream_t s);
void release_ws(prag_gpu_index* ix, Workspace* w, cudaStream_t s);
int ws_reserve(Workspace* w, size_t bytes, cudaStream_t s);
int ws_reserve_stage(Workspace* w, size_t bytes, cudaStream_t s);
int ws_reserve_host(Workspace* w, size_t bytes);
int validate(const prag_gpu_index* ix, uint32_t nprobe, uint32_t k);
int run_coarse(const prag_gpu_index* ix, const float* dq, uint32_t nq, uint32_t nprobe, float* coarse,
               uint32_t* probe, float* probe_dist, uint32_t* pkey, uint64_t* ptie, cudaStream_t s,
               Workspace* prof_ws = nullptr);
// One pass over nq device-resident queries into device outputs, on stream s.
int search_pass(prag_gpu_index* ix, Workspace* w, const float* dq, uint32_t nq, uint32_t nprobe, uint32_t k,
                uint64_t* o_ids, float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s,
                prag_gpu_timings* tm, bool rerank);
// Queries per pass: a pure function of the WHOLE index's list sizes and the
// shape, so every rank of a distributed index makes the same passes.
uint32_t pass_chunk(const prag_gpu_index* ix, uint32_t nq, uint32_t nprobe, uint32_t k, bool rerank);
int do_search(prag_gpu_index* ix, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t k,
              uint64_t* out_ids, float* out_dist, uint32_t* out_count, uint64_t* out_scanned, cudaStream_t s,
              bool rerank = false, bool all_device = false);
bool uses_fast_path(const prag_gpu_index* ix, uint32_t k, bool rerank);
std::vector<uint64_t> prefix_desc(const std::vector<uint64_t>& sizes);
int ws_reserve_x(Workspace* w, size_t bytes, cudaStream_t s);
void free_ws(Workspace* w);

// ------------------------------------------------ list sharding (shard.cu)
struct GroupPlan;
// Group handle: every shard's pass on its own device/stream, then the fused
// peer-memory gather + merge on the root stream s. With `plan` the shard
// passes replay that plan's captured graphs and dedicated workspaces.
int group_pass(prag_gpu_index* g, Workspace* wg, const float* dq, uint32_t nq, uint32_t nprobe, uint32_t k,
               uint64_t* o_ids, float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s, bool rerank,
               GroupPlan* plan);
// Distributed shard (NCCL comm attached): local pass into the rank's top-k
// block, ncclAllGather of the blocks on s, merge on every rank.
int dist_pass(prag_gpu_index* ix, Workspace* w, const float* dq, uint32_t nq, uint32_t nprobe, uint32_t k,
              uint64_t* o_ids, float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s,
              prag_gpu_timings* tm, bool rerank);
int group_plan_create(prag_gpu_index* g, const float* dq, uint32_t nq, uint32_t nprobe, uint32_t k, uint64_t* o_ids,
                      float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s, GroupPlan** out);
int group_plan_launch(prag_gpu_index* g, GroupPlan* p, cudaStream_t s);
void group_plan_free(prag_gpu_index* g, GroupPlan* p);
void free_group(prag_gpu_index* g);
// synthetic index (capi.cu): rank `rank` of `world` (world 1: the whole index)
int build_synthetic(uint32_t nlist, uint32_t d, uint32_t nsq, uint64_t ntotal, uint64_t seed, double sigma,
                    const float* centroids, const float* codewords, int rank, int world, int device,
                    prag_gpu_index** out);

}  // namespace pg

struct prag_gpu_plan {
    prag_gpu_index* ix = nullptr;
    pg::Workspace* w = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    pg::GroupPlan* group = nullptr;  // group handle: per-shard graphs + the root merge
};
