// shard.cu -- list-sharded search across GPUs.
//
// IVF lists are independent and a candidate's distance depends only on
// (query, its list, its code), so the global top-k is the exact top-k of the
// union of the per-shard top-k lists, ordered by (distance, chunk id)
// (annindex.hpp:54-60, :313). Every shard holds the replicated centroids and
// codebook, computes the identical probe set, and scans only the probed lists
// it owns (K1-K4 of capi.cu's search_pass). Two ways to put shards together:
//
//  * group handle (one process, several devices): every shard's pass runs on
//    its own device and stream; then ONE kernel on the root device reads each
//    shard's k-list block straight from that GPU's memory over NVLink (peer
//    access) and merges -- the gather fused into the merge, no staging copy.
//  * distributed shard (one process per GPU): the rank's block goes through
//    one ncclAllGather on the search stream, then the same merge kernel runs
//    on every rank over the gathered blocks. NCCL is resolved with dlopen, so
//    the library has no link-time NCCL dependency and shares the copy torch
//    (or the caller) already loaded.
//
// The per-shard block of one pass: ids [nq][k] u64 | dist [nq][k] f32 |
// count [nq] u32 | scanned [nq] u64, at fixed 256-byte-aligned offsets.
#include <dlfcn.h>
#include <nccl.h>  // types and enums only; every symbol comes from dlsym

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>

#include "internal.h"

struct prag_gpu_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, device = 0;
};

namespace pg {

// ------------------------------------------------------------ NCCL (dlopen)
namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // RTLD_NOLOAD first: the NCCL this process already mapped (torch's)
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllGather || !api.GetErrorString)
            api.error = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

int nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return PRAG_GPU_OK;
    set_error(std::string("NCCL error in ") + what + ": " + nccl().GetErrorString(r));
    return PRAG_GPU_NCCL;
}

int nccl_ready() {
    if (!nccl().error.empty()) {
        set_error(nccl().error);
        return PRAG_GPU_NCCL;
    }
    return PRAG_GPU_OK;
}

// ------------------------------------------------------- per-shard blocks
struct PartLayout {
    size_t ids, dist, count, scanned, bytes;
};

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

PartLayout part_layout(uint32_t nq, uint32_t k) {
    PartLayout L;
    L.ids = 0;
    L.dist = align256(size_t(nq) * k * 8);
    L.count = align256(L.dist + size_t(nq) * k * 4);
    L.scanned = align256(L.count + size_t(nq) * 4);
    L.bytes = align256(L.scanned + size_t(nq) * 8);
    return L;
}

constexpr int kMaxParts = 32;

struct PartsArg {
    const unsigned char* base[kMaxParts];  // block of part p (any device the root can read)
};

__device__ __forceinline__ uint32_t ord_key(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// One warp per query: lane p holds the head of part p's list (sorted by
// (distance, chunk id), count[p][q] entries); k rounds of "smallest (key, id)
// among the heads" produce the exact merged list. Part blocks are read where
// they live: over NVLink for peer shards.
__global__ void __launch_bounds__(256) merge_parts_kernel(const PartsArg parts, uint32_t nparts, uint32_t nq,
                                                          uint32_t k, size_t o_dist, size_t o_count,
                                                          size_t o_scanned, uint64_t* __restrict__ out_ids,
                                                          float* __restrict__ out_dist,
                                                          uint32_t* __restrict__ out_count,
                                                          uint64_t* __restrict__ out_scanned) {
    const uint32_t lane = threadIdx.x & 31, q = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (q >= nq) return;
    const bool own = lane < nparts;
    const unsigned char* b = own ? parts.base[lane] : nullptr;
    const uint64_t* ids = own ? reinterpret_cast<const uint64_t*>(b) + size_t(q) * k : nullptr;
    const float* dist = own ? reinterpret_cast<const float*>(b + o_dist) + size_t(q) * k : nullptr;
    const uint32_t cnt = own ? min(reinterpret_cast<const uint32_t*>(b + o_count)[q], k) : 0u;
    uint64_t sc = own ? reinterpret_cast<const uint64_t*>(b + o_scanned)[q] : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
    uint32_t h = 0;
    float hd = cnt ? dist[0] : 0.0f;
    uint32_t hk = cnt ? ord_key(hd) : 0xffffffffu;
    uint64_t hid = cnt ? ids[0] : ~0ull;
    uint32_t r = 0;
    for (; r < k; ++r) {
        const uint32_t kmin = __reduce_min_sync(0xffffffffu, hk);
        if (kmin == 0xffffffffu) break;
        uint64_t cid = hk == kmin ? hid : ~0ull;  // exact distance tie: lowest chunk id
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const uint64_t x = __shfl_xor_sync(0xffffffffu, cid, o);
            cid = x < cid ? x : cid;
        }
        const unsigned win = __ballot_sync(0xffffffffu, hk == kmin && hid == cid);
        if (int(lane) == __ffs(win) - 1) {
            out_ids[size_t(q) * k + r] = hid;
            out_dist[size_t(q) * k + r] = hd;
            if (++h < cnt) {
                hd = dist[h];
                hk = ord_key(hd);
                hid = ids[h];
            } else {
                hk = 0xffffffffu;
                hid = ~0ull;
            }
        }
    }
    if (lane == 0) {
        out_count[q] = r;
        if (out_scanned) out_scanned[q] = sc;
    }
}

int launch_merge_parts(const PartsArg& a, uint32_t nparts, uint32_t nq, uint32_t k, const PartLayout& L,
                       uint64_t* o_ids, float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s) {
    merge_parts_kernel<<<(nq + 7) / 8, 256, 0, s>>>(a, nparts, nq, k, L.dist, L.count, L.scanned, o_ids, o_dist,
                                                    o_count, o_scanned);
    PG_CUDA(cudaGetLastError());
    return PRAG_GPU_OK;
}

Workspace* new_ws(int device) {
    auto* w = new Workspace();
    w->device = device;
    cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&w->host_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&w->xev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&w->xev2, cudaEventDisableTiming);
    return w;
}

}  // namespace

// --------------------------------------------------------- group handle
struct GroupPlan {
    uint32_t nq = 0, nprobe = 0, k = 0;
    const float* dq = nullptr;  // root-device query buffer the plan reads
    uint64_t* o_ids = nullptr;
    float* o_dist = nullptr;
    uint32_t* o_count = nullptr;
    uint64_t* o_scanned = nullptr;
    Workspace* wg = nullptr;                  // root: gathered blocks of non-peer shards
    std::vector<Workspace*> ws;               // per shard: scratch, query copy, its block
    std::vector<cudaGraphExec_t> exec;        // per shard: its captured K1-K4 pass
};

// Queries for shard r: the root buffer itself on the root device, else a
// copy into the shard's staging (98 KiB at nq 64, d 384) on the shard stream.
static int shard_queries(prag_gpu_index* g, int r, Workspace* w, const float* dq, uint32_t nq, cudaStream_t st,
                         const float** out) {
    const prag_gpu_index* sh = g->shards[r];
    if (sh->device == g->device) {
        *out = dq;
        return PRAG_GPU_OK;
    }
    const size_t qb = size_t(nq) * g->dev.d * 4;
    PG_TRY(ws_reserve_stage(w, qb, st));
    PG_CUDA(cudaMemcpyPeerAsync(w->stage, sh->device, dq, g->device, qb, st));
    *out = static_cast<const float*>(w->stage);
    return PRAG_GPU_OK;
}

int group_pass(prag_gpu_index* g, Workspace* wg, const float* dq, uint32_t nq, uint32_t nprobe, uint32_t k,
               uint64_t* o_ids, float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s, bool rerank,
               GroupPlan* plan) {
    const int n = int(g->shards.size());
    const PartLayout L = part_layout(nq, k);
    std::vector<Workspace*> ws(n, nullptr);
    // the root stream's work so far (queries) is what every shard waits for
    PG_CUDA(cudaEventRecord(wg->xev, s));
    int rc = PRAG_GPU_OK;
    for (int r = 0; r < n && rc == PRAG_GPU_OK; ++r) {
        prag_gpu_index* sh = g->shards[r];
        DeviceGuard dg(sh->device);
        cudaStream_t st = g->shard_streams[r];
        ws[r] = plan ? plan->ws[r] : acquire_ws(sh, st);
        Workspace* w = ws[r];
        PG_CUDA(cudaStreamWaitEvent(st, wg->xev, 0));
        const float* q = nullptr;
        if ((rc = shard_queries(g, r, w, dq, nq, st, &q))) break;
        if (plan) {
            PG_CUDA(cudaGraphLaunch(plan->exec[r], st));
        } else {
            if ((rc = ws_reserve_x(w, L.bytes, st))) break;
            unsigned char* blk = static_cast<unsigned char*>(w->xbuf);
            prag_gpu_timings tm{};
            const bool prof = r == 0 && sh->profiling;
            rc = search_pass(sh, w, q, nq, nprobe, k, reinterpret_cast<uint64_t*>(blk + L.ids),
                             reinterpret_cast<float*>(blk + L.dist), reinterpret_cast<uint32_t*>(blk + L.count),
                             reinterpret_cast<uint64_t*>(blk + L.scanned), st, prof ? &tm : nullptr, rerank);
            if (prof && rc == PRAG_GPU_OK) {
                std::lock_guard<std::mutex> lk(sh->mu);
                sh->last = tm;
            }
            if (rc) break;
        }
        PG_CUDA(cudaEventRecord(w->xev, st));
    }
    // fused gather + merge on the root: blocks of peer-reachable shards are
    // read in place; the others are copied next to the root first
    PartsArg a{};
    if (rc == PRAG_GPU_OK) {
        size_t far = 0;
        for (int r = 0; r < n; ++r)
            if (!g->peer_direct[r]) ++far;
        if (far) rc = ws_reserve_x(wg, far * L.bytes, s);
        size_t fi = 0;
        for (int r = 0; r < n && rc == PRAG_GPU_OK; ++r) {
            PG_CUDA(cudaStreamWaitEvent(s, ws[r]->xev, 0));
            const unsigned char* blk = static_cast<const unsigned char*>(ws[r]->xbuf);
            if (!g->peer_direct[r]) {
                unsigned char* dst = static_cast<unsigned char*>(wg->xbuf) + (fi++) * L.bytes;
                PG_CUDA(cudaMemcpyPeerAsync(dst, g->device, blk, g->shards[r]->device, L.bytes, s));
                blk = dst;
            }
            a.base[r] = blk;
        }
    }
    if (rc == PRAG_GPU_OK) rc = launch_merge_parts(a, uint32_t(n), nq, k, L, o_ids, o_dist, o_count, o_scanned, s);
    // the shards' scratch and blocks are free again once the merge has read them
    cudaEventRecord(wg->xev2, s);
    for (int r = 0; r < n; ++r) {
        if (!ws[r]) continue;
        DeviceGuard dg(g->shards[r]->device);
        cudaStreamWaitEvent(g->shard_streams[r], wg->xev2, 0);
        if (!plan) release_ws(g->shards[r], ws[r], g->shard_streams[r]);
    }
    return rc;
}

int group_plan_create(prag_gpu_index* g, const float* dq, uint32_t nq, uint32_t nprobe, uint32_t k, uint64_t* o_ids,
                      float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s, GroupPlan** out) {
    auto p = std::make_unique<GroupPlan>();
    p->nq = nq;
    p->nprobe = nprobe;
    p->k = k;
    p->dq = dq;
    p->o_ids = o_ids;
    p->o_dist = o_dist;
    p->o_count = o_count;
    p->o_scanned = o_scanned;
    struct Cleanup {
        prag_gpu_index* g;
        GroupPlan* p;
        ~Cleanup() {
            if (p) group_plan_free(g, p);
        }
    } cleanup{g, p.get()};
    p->wg = new_ws(g->device);
    const int n = int(g->shards.size());
    const PartLayout L = part_layout(nq, k);
    p->ws.assign(n, nullptr);
    p->exec.assign(n, nullptr);
    for (int r = 0; r < n; ++r) {
        prag_gpu_index* sh = g->shards[r];
        DeviceGuard dg(sh->device);
        cudaStream_t st = g->shard_streams[r];
        p->ws[r] = new_ws(sh->device);
        Workspace* w = p->ws[r];
        // queries the shard's pass reads (its own copy off the root device)
        const float* q = dq;
        if (sh->device != g->device) {
            PG_TRY(ws_reserve_stage(w, size_t(nq) * g->dev.d * 4, st));
            q = static_cast<const float*>(w->stage);
        }
        PG_TRY(ws_reserve_x(w, L.bytes, st));
        unsigned char* blk = static_cast<unsigned char*>(w->xbuf);
        uint64_t* bi = reinterpret_cast<uint64_t*>(blk + L.ids);
        float* bd = reinterpret_cast<float*>(blk + L.dist);
        uint32_t* bc = reinterpret_cast<uint32_t*>(blk + L.count);
        uint64_t* bs = reinterpret_cast<uint64_t*>(blk + L.scanned);
        // size the workspace with one ordinary pass, then capture the same pass
        PG_CUDA(cudaMemsetAsync(w->xbuf, 0, L.bytes, st));
        if (sh->device != g->device)
            PG_CUDA(cudaMemcpyPeerAsync(w->stage, sh->device, dq, g->device, size_t(nq) * g->dev.d * 4, st));
        PG_TRY(search_pass(sh, w, q, nq, nprobe, k, bi, bd, bc, bs, st, nullptr, false));
        PG_CUDA(cudaStreamSynchronize(st));
        // (shard streams are private non-blocking streams: capturable)
        PG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        const int rc = search_pass(sh, w, q, nq, nprobe, k, bi, bd, bc, bs, st, nullptr, false);
        cudaGraph_t graph = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(st, &graph);
        if (rc != PRAG_GPU_OK) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        PG_CUDA(ce);
        const cudaError_t ie = cudaGraphInstantiate(&p->exec[r], graph, 0);
        cudaGraphDestroy(graph);
        PG_CUDA(ie);
    }
    {
        size_t far = 0;
        for (int r = 0; r < n; ++r)
            if (!g->peer_direct[r]) ++far;
        if (far) PG_TRY(ws_reserve_x(p->wg, far * L.bytes, s));
    }
    cleanup.p = nullptr;
    *out = p.release();
    return PRAG_GPU_OK;
}

int group_plan_launch(prag_gpu_index* g, GroupPlan* p, cudaStream_t s) {
    DeviceGuard dg(g->device);
    return group_pass(g, p->wg, p->dq, p->nq, p->nprobe, p->k, p->o_ids, p->o_dist, p->o_count, p->o_scanned, s,
                      false, p);
}

void group_plan_free(prag_gpu_index* g, GroupPlan* p) {
    if (!p) return;
    for (size_t r = 0; r < p->ws.size(); ++r) {
        DeviceGuard dg(g->shards[r]->device);
        cudaDeviceSynchronize();
        if (r < p->exec.size() && p->exec[r]) cudaGraphExecDestroy(p->exec[r]);
        free_ws(p->ws[r]);
    }
    if (p->wg) {
        DeviceGuard dg(g->device);
        cudaDeviceSynchronize();
        free_ws(p->wg);
    }
    delete p;
}

void free_group(prag_gpu_index* g) {
    for (size_t r = 0; r < g->shards.size(); ++r) {
        {
            DeviceGuard dg(g->shards[r]->device);
            cudaStreamSynchronize(g->shard_streams[r]);
            cudaStreamDestroy(g->shard_streams[r]);
        }
        prag_gpu_index_free(g->shards[r]);
    }
    g->shards.clear();
    g->shard_streams.clear();
    DeviceGuard dg(g->device);
    cudaDeviceSynchronize();
    for (Workspace* w : g->pool) free_ws(w);
    g->pool.clear();
}

// Builds the group handle over owned shards (ranks 0..n-1 of world n).
static int make_group(std::vector<prag_gpu_index*>& shards, prag_gpu_index** out) {
    const int n = int(shards.size());
    auto g = std::make_unique<prag_gpu_index>();
    const prag_gpu_index* s0 = shards[0];
    g->device = s0->device;
    g->ntotal_global = s0->ntotal_global;
    g->dev.nlist = s0->dev.nlist;
    g->dev.d = s0->dev.d;
    g->dev.nsq = s0->dev.nsq;
    g->dev.sub_dim = s0->dev.sub_dim;
    g->dev.code_layout = s0->dev.code_layout;
    g->dev.plain_codes = s0->dev.plain_codes;
    g->dev.tc_ok = s0->dev.tc_ok;
    g->scan_path = s0->scan_path;
    g->coarse_path = s0->coarse_path;
    g->host_list_len.assign(g->dev.nlist, 0);
    for (const prag_gpu_index* sh : shards) {
        for (uint32_t l = 0; l < g->dev.nlist; ++l) g->host_list_len[l] += sh->host_list_len[l];
        g->dev.ntotal += sh->dev.ntotal;
        g->dev.max_list_len = std::max(g->dev.max_list_len, sh->dev.max_list_len);
    }
    g->top_prefix = prefix_desc(g->host_list_len);
    g->global_top_prefix = g->top_prefix;
    g->shard_world = 1;  // the group is the whole index
    g->peer_direct.assign(n, 1);
    g->shard_streams.assign(n, nullptr);
    for (int r = 0; r < n; ++r) {
        const int dv = shards[r]->device;
        {
            DeviceGuard dg(dv);
            PG_CUDA(cudaStreamCreateWithFlags(&g->shard_streams[r], cudaStreamNonBlocking));
        }
        if (dv == g->device) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, g->device, dv);
        if (can) {  // the root's merge kernel reads shard dv's block in place
            DeviceGuard dg(g->device);
            const cudaError_t e = cudaDeviceEnablePeerAccess(dv, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) can = 0;
            cudaGetLastError();
        }
        g->peer_direct[r] = uint8_t(can != 0);
    }
    g->shards = shards;
    shards.clear();
    *out = g.release();
    return PRAG_GPU_OK;
}

// Splits a host index into n shards (plan_shard_ranges: whole lists by LPT,
// the largest striped) uploaded to devices[r], grouped.
static int group_from_host(const HostIndex& h, const int* devices, int n, prag_gpu_index** out) {
    if (n > kMaxParts) {
        set_error("sharded index: at most " + std::to_string(kMaxParts) + " shards");
        return PRAG_GPU_CONFIG;
    }
    for (int r = 0; r < n; ++r) PG_TRY(require_device(devices[r]));
    const uint32_t nl = h.nlist;
    std::vector<uint64_t> sizes(nl);
    for (uint32_t l = 0; l < nl; ++l) sizes[l] = h.list_off[l + 1] - h.list_off[l];
    std::vector<uint64_t> rb(nl), re(nl);
    std::vector<prag_gpu_index*> shards;
    struct Free {
        std::vector<prag_gpu_index*>& v;
        ~Free() {
            for (auto* p : v) prag_gpu_index_free(p);
        }
    } guard{shards};
    for (int r = 0; r < n; ++r) {
        plan_shard_ranges(sizes.data(), nl, uint32_t(n), uint32_t(r), rb.data(), re.data());
        HostIndex hr;
        hr.nlist = h.nlist;
        hr.d = h.d;
        hr.nsq = h.nsq;
        hr.sub_dim = h.sub_dim;
        hr.centroids = h.centroids;
        hr.codewords = h.codewords;
        hr.ntotal_global = h.ntotal_global ? h.ntotal_global : h.ids.size();
        hr.list_off.assign(size_t(nl) + 1, 0);
        for (uint32_t l = 0; l < nl; ++l) {
            const uint64_t b = h.list_off[l] + rb[l], len = re[l] - rb[l];  // whole list or a stripe
            if (len) {
                hr.ids.insert(hr.ids.end(), h.ids.begin() + b, h.ids.begin() + b + len);
                hr.codes.insert(hr.codes.end(), h.codes.begin() + b * h.nsq, h.codes.begin() + (b + len) * h.nsq);
            }
            hr.list_off[l + 1] = hr.list_off[l] + len;
        }
        auto ix = std::make_unique<prag_gpu_index>();
        ix->shard_rank = r;
        ix->shard_world = n;
        ix->global_top_prefix = prefix_desc(sizes);
        prag_gpu_index* p = nullptr;
        PG_TRY(finish_load(ix, hr, devices[r], &p));
        shards.push_back(p);
    }
    return make_group(shards, out);
}

// ------------------------------------------------------- distributed rank
int dist_pass(prag_gpu_index* ix, Workspace* w, const float* dq, uint32_t nq, uint32_t nprobe, uint32_t k,
              uint64_t* o_ids, float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s,
              prag_gpu_timings* tm, bool rerank) {
    PG_TRY(nccl_ready());
    const prag_gpu_comm* c = ix->comm;
    const PartLayout L = part_layout(nq, k);
    // [own block][world gathered blocks]
    PG_TRY(ws_reserve_x(w, L.bytes * (size_t(c->world) + 1), s));
    unsigned char* mine = static_cast<unsigned char*>(w->xbuf);
    unsigned char* all = mine + L.bytes;
    PG_TRY(search_pass(ix, w, dq, nq, nprobe, k, reinterpret_cast<uint64_t*>(mine + L.ids),
                       reinterpret_cast<float*>(mine + L.dist), reinterpret_cast<uint32_t*>(mine + L.count),
                       reinterpret_cast<uint64_t*>(mine + L.scanned), s, tm, rerank));
    PG_TRY(nccl_check(nccl().AllGather(mine, all, L.bytes, ncclUint8, c->comm, s), "ncclAllGather"));
    PartsArg a{};
    for (int r = 0; r < c->world; ++r) a.base[r] = all + size_t(r) * L.bytes;
    return launch_merge_parts(a, uint32_t(c->world), nq, k, L, o_ids, o_dist, o_count, o_scanned, s);
}

}  // namespace pg

using namespace pg;

extern "C" {

int prag_gpu_index_group(prag_gpu_index* const* shards, int n, prag_gpu_index** out) {
    PG_API_BEGIN
    if (!out || !shards || n < 1) {
        set_error("group: need >= 1 shard");
        return PRAG_GPU_CONFIG;
    }
    *out = nullptr;
    if (n > kMaxParts) {
        set_error("group: at most " + std::to_string(kMaxParts) + " shards");
        return PRAG_GPU_CONFIG;
    }
    std::vector<uint8_t> seen(n, 0);
    for (int r = 0; r < n; ++r) {
        const prag_gpu_index* sh = shards[r];
        if (!sh || sh->is_group() || sh->comm) {
            set_error("group: every element must be a plain shard handle");
            return PRAG_GPU_CONFIG;
        }
        if (sh->shard_world != n || sh->shard_rank < 0 || sh->shard_rank >= n || seen[sh->shard_rank]) {
            set_error("group: shards must be ranks 0..n-1 of one world of n");
            return PRAG_GPU_CONFIG;
        }
        seen[sh->shard_rank] = 1;
        if (sh->dev.nlist != shards[0]->dev.nlist || sh->dev.d != shards[0]->dev.d ||
            sh->dev.nsq != shards[0]->dev.nsq || sh->ntotal_global != shards[0]->ntotal_global) {
            set_error("group: shards of different indexes");
            return PRAG_GPU_CONFIG;
        }
    }
    std::vector<prag_gpu_index*> v(n);
    for (int r = 0; r < n; ++r) v[shards[r]->shard_rank] = shards[r];  // root = rank 0
    return make_group(v, out);
    PG_API_END
}

int prag_gpu_index_load_sharded(const char* path, const int* devices, int n, prag_gpu_index** out) {
    PG_API_BEGIN
    if (!out || !path || !devices || n < 1) {
        set_error("load_sharded: need a path and >= 1 device");
        return PRAG_GPU_CONFIG;
    }
    *out = nullptr;
    // one read of the file; each shard keeps the lists LPT gives it
    HostIndex h;
    PG_TRY(read_pragix01(path, h, nullptr));
    return group_from_host(h, devices, n, out);
    PG_API_END
}

int prag_gpu_index_from_host_sharded(uint32_t nlist, uint32_t d, uint32_t nsq, const float* centroids,
                                     const float* codewords, const uint64_t* list_off, const uint64_t* ids,
                                     const uint8_t* codes, const int* devices, int n, prag_gpu_index** out) {
    PG_API_BEGIN
    if (!out || !devices || n < 1 || !centroids || !codewords || !list_off) {
        set_error("from_host_sharded: null argument or no device");
        return PRAG_GPU_CONFIG;
    }
    *out = nullptr;
    if (nsq == 0 || d % nsq != 0) {
        set_error("invalid n_subquantizers");
        return PRAG_GPU_CONFIG;
    }
    for (uint32_t l = 0; l < nlist; ++l)
        if (list_off[l + 1] < list_off[l]) {
            set_error("list_off must be non-decreasing");
            return PRAG_GPU_CONFIG;
        }
    HostIndex h;
    h.nlist = nlist;
    h.d = d;
    h.nsq = nsq;
    h.sub_dim = d / nsq;
    h.centroids.assign(centroids, centroids + size_t(nlist) * d);
    h.codewords.assign(codewords, codewords + size_t(nsq) * 256 * (d / nsq));
    h.list_off.assign(list_off, list_off + nlist + 1);
    const uint64_t total = list_off[nlist];
    h.ids.assign(ids, ids + total);
    h.codes.assign(codes, codes + total * nsq);
    h.ntotal_global = total;
    return group_from_host(h, devices, n, out);
    PG_API_END
}

int prag_gpu_comm_unique_id(uint8_t out_id[128]) {
    PG_API_BEGIN
    if (!out_id) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    PG_TRY(nccl_ready());
    ncclUniqueId id;
    PG_TRY(nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId"));
    static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out_id, id.internal, 128);
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_comm_init(const uint8_t id_bytes[128], int world, int rank, int device, prag_gpu_comm** out) {
    PG_API_BEGIN
    if (!out || !id_bytes || world < 1 || rank < 0 || rank >= world) {
        set_error("comm_init: invalid arguments");
        return PRAG_GPU_CONFIG;
    }
    *out = nullptr;
    if (world > kMaxParts) {
        set_error("comm_init: at most " + std::to_string(kMaxParts) + " ranks");
        return PRAG_GPU_CONFIG;
    }
    PG_TRY(require_device(device));
    PG_TRY(nccl_ready());
    DeviceGuard g(device);
    ncclUniqueId id;
    std::memcpy(id.internal, id_bytes, 128);
    auto c = std::make_unique<prag_gpu_comm>();
    c->rank = rank;
    c->world = world;
    c->device = device;
    PG_TRY(nccl_check(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank"));
    *out = c.release();
    return PRAG_GPU_OK;
    PG_API_END
}

void prag_gpu_comm_free(prag_gpu_comm* c) {
    if (!c) return;
    if (c->comm && nccl().CommDestroy) {
        DeviceGuard g(c->device);
        nccl().CommDestroy(c->comm);
    }
    delete c;
}

int prag_gpu_index_attach_comm(prag_gpu_index* ix, prag_gpu_comm* c) {
    PG_API_BEGIN
    if (!ix || ix->is_group()) {
        set_error("attach_comm: need a shard handle");
        return PRAG_GPU_CONFIG;
    }
    if (c && (c->world != ix->shard_world || c->rank != ix->shard_rank || c->device != ix->device)) {
        set_error("attach_comm: comm rank/world/device must match the shard's (rank " +
                  std::to_string(ix->shard_rank) + " of " + std::to_string(ix->shard_world) + " on device " +
                  std::to_string(ix->device) + ")");
        return PRAG_GPU_CONFIG;
    }
    ix->comm = c;
    return PRAG_GPU_OK;
    PG_API_END
}

}  // extern "C"
