// capi.cu -- C ABI of the B200 IVF-PQ search path (include/prag_gpu.h):
// index lifecycle (PRAGIX01 -> HBM layout), search orchestration on a CUDA
// stream, shard planning/merge, and the GPU-fed performance model.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>

#include <map>

#include "internal.h"

namespace pg {

static thread_local std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }

// (orchestration helpers: declared in internal.h, shared with shard.cu)


int require_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        set_error("no CUDA device visible: the prag_gpu search path has no CPU fallback");
        return PRAG_GPU_NO_DEVICE;
    }
    if (device < 0 || device >= n) {
        set_error("CUDA device " + std::to_string(device) + " out of range (" + std::to_string(n) + " visible)");
        return PRAG_GPU_CONFIG;
    }
    return PRAG_GPU_OK;
}


// SMs the persistent search kernels size their grids to: the device's, or
// the index's budget (prag_gpu_set_sm_budget) when retrieval shares the GPU
// with other work pinned to the remaining SMs (config E).
int search_sms(const prag_gpu_index* ix) {
    const int all = sm_count(ix->device);
    return ix->sm_budget > 0 ? std::min(all, ix->sm_budget) : all;
}

int sm_count(int device) {
    static std::atomic<int> cache[64];
    if (device < 0 || device >= 64) {
        int n = 148;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
        return n;
    }
    int n = cache[device].load(std::memory_order_relaxed);
    if (n == 0) {
        n = 148;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
        cache[device].store(n, std::memory_order_relaxed);
    }
    return n;
}

cudaError_t ensure_smem(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{kernel, dev}];
    if (have >= bytes && have) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    if (e == cudaSuccess) have = bytes;
    return e;
}
// (orchestration helpers: declared in internal.h, shared with shard.cu)

bool is_device_ptr(const void* p) {
    if (p == nullptr) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool is_pinned_host(const void* p) {
    cudaPointerAttributes a{};
    if (p == nullptr || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

template <typename T>
int dmalloc(T** p, size_t n, uint64_t* acct) {
    size_t bytes = std::max<size_t>(n * sizeof(T), 16);
    PG_CUDA(cudaMalloc(reinterpret_cast<void**>(p), bytes));
    if (acct) *acct += bytes;
    return PRAG_GPU_OK;
}

void free_device_index(DeviceIndex& d) {
    cudaFree(d.centroids);
    cudaFree(d.centroidsT);
    cudaFree(d.centroids4);
    cudaFree(d.codewordsT);
    cudaFree(d.list_off);
    cudaFree(d.list_len);
    cudaFree(d.ids);
    cudaFree(d.codes);
    cudaFree(d.codewords);
    cudaFree(d.skew_off);
    cudaFree(d.skew_codes);
    cudaFree(d.cent_tc);
    cudaFree(d.cent_norm);
    d = DeviceIndex{};
}

// Host SoA (reference logical layout) -> HBM layout:
//  centroids [nlist][d] and transposed [d][nlist]; codewords transposed to
//  [nsq][sub_dim][256] so a warp building the ADC table reads consecutive
//  codes; lists padded to multiples of kListPad entries, 16-byte aligned.
int upload(prag_gpu_index* ix, const HostIndex& h) {
    DeviceIndex& d = ix->dev;
    d.nlist = h.nlist;
    d.d = h.d;
    d.nsq = h.nsq;
    d.sub_dim = h.sub_dim;
    const uint32_t nl = h.nlist;
    std::vector<uint64_t> off(size_t(nl) + 1, 0);
    std::vector<uint32_t> len(nl);
    ix->host_list_len.assign(nl, 0);
    uint32_t maxlen = 0;
    for (uint32_t l = 0; l < nl; ++l) {
        uint64_t n = h.list_off[l + 1] - h.list_off[l];
        if (n >= (1ull << 32)) {
            set_error("list " + std::to_string(l) + " exceeds 2^32 entries");
            return PRAG_GPU_CONFIG;
        }
        len[l] = uint32_t(n);
        ix->host_list_len[l] = n;
        maxlen = std::max(maxlen, len[l]);
        off[l + 1] = off[l] + (n + kListPad - 1) / kListPad * kListPad;
    }
    d.ntotal = h.list_off[nl];
    d.npadded = off[nl];
    d.max_list_len = maxlen;
    if (d.npadded >= (1ull << 32)) {
        set_error("more than 2^32 resident entries on one device; shard the index");
        return PRAG_GPU_CONFIG;
    }
    ix->top_prefix = prefix_desc(ix->host_list_len);
    if (ix->global_top_prefix.empty()) ix->global_top_prefix = ix->top_prefix;

    uint64_t* acct = &ix->device_bytes;
    PG_TRY(dmalloc(&d.centroids, size_t(nl) * h.d, acct));
    PG_TRY(dmalloc(&d.centroidsT, size_t(nl) * h.d, acct));
    PG_TRY(dmalloc(&d.codewordsT, size_t(h.nsq) * 256 * h.sub_dim, acct));
    PG_TRY(dmalloc(&d.list_off, size_t(nl) + 1, acct));
    PG_TRY(dmalloc(&d.list_len, nl, acct));
    PG_TRY(dmalloc(&d.ids, d.npadded, acct));
    // m = 32 / 64: the lane-skewed tiles are the only copy of the codes in
    // HBM (the generic path gathers from them too); other m: plain [slot][m]
    const bool skew_only = (h.nsq == 32 || h.nsq == 64) && h.sub_dim <= 16;
    if (!skew_only) PG_TRY(dmalloc(&d.codes, d.npadded * h.nsq, acct));
    d.plain_codes = !skew_only;

    PG_CUDA(cudaMemcpy(d.centroids, h.centroids.data(), h.centroids.size() * 4, cudaMemcpyHostToDevice));
    {
        std::vector<float> t(size_t(nl) * h.d);
        for (uint32_t c = 0; c < nl; ++c)
            for (uint32_t j = 0; j < h.d; ++j) t[size_t(j) * nl + c] = h.centroids[size_t(c) * h.d + j];
        PG_CUDA(cudaMemcpy(d.centroidsT, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
    }
    {
        std::vector<float> t(size_t(h.nsq) * 256 * h.sub_dim);
        for (uint32_t s = 0; s < h.nsq; ++s)
            for (uint32_t c = 0; c < 256; ++c)
                for (uint32_t j = 0; j < h.sub_dim; ++j)
                    t[(size_t(s) * h.sub_dim + j) * 256 + c] = h.codewords[(size_t(s) * 256 + c) * h.sub_dim + j];
        PG_CUDA(cudaMemcpy(d.codewordsT, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
    }
    if (h.d % 4 == 0) {
        std::vector<float> t(size_t(nl) * h.d);
        for (uint32_t c = 0; c < nl; ++c)
            for (uint32_t j = 0; j < h.d; ++j) t[(size_t(j / 4) * nl + c) * 4 + (j % 4)] = h.centroids[size_t(c) * h.d + j];
        PG_TRY(dmalloc(&d.centroids4, t.size(), acct));
        PG_CUDA(cudaMemcpy(d.centroids4, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
    }
    PG_CUDA(cudaMemcpy(d.list_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
    PG_CUDA(cudaMemcpy(d.list_len, len.data(), len.size() * 4, cudaMemcpyHostToDevice));
    {
        // padded ids (pad = ~0) and codes (pad = 0), uploaded list by list group
        std::vector<uint64_t> pid(d.npadded, ~0ull);
        std::vector<uint8_t> pcode(d.codes ? d.npadded * h.nsq : 0, 0);
        for (uint32_t l = 0; l < nl; ++l) {
            const uint64_t src = h.list_off[l], n = len[l];
            std::memcpy(&pid[off[l]], &h.ids[src], n * 8);
            if (d.codes) std::memcpy(&pcode[off[l] * h.nsq], &h.codes[src * h.nsq], n * h.nsq);
        }
        PG_CUDA(cudaMemcpy(d.ids, pid.data(), pid.size() * 8, cudaMemcpyHostToDevice));
        if (d.codes) PG_CUDA(cudaMemcpy(d.codes, pcode.data(), pcode.size(), cudaMemcpyHostToDevice));
    }
    d.code_layout = 0;
    PG_TRY(dmalloc(&d.codewords, h.codewords.size(), acct));
    PG_CUDA(cudaMemcpy(d.codewords, h.codewords.data(), h.codewords.size() * 4, cudaMemcpyHostToDevice));
    if (skew_only) {
        std::vector<uint64_t> soff;
        std::vector<uint8_t> scodes;
        build_skew_layout(h, h.nsq, soff, scodes);
        PG_TRY(dmalloc(&d.skew_off, soff.size(), acct));
        PG_TRY(dmalloc(&d.skew_codes, scodes.size(), acct));
        PG_CUDA(cudaMemcpy(d.skew_off, soff.data(), soff.size() * 8, cudaMemcpyHostToDevice));
        PG_CUDA(cudaMemcpy(d.skew_codes, scodes.data(), scodes.size(), cudaMemcpyHostToDevice));
        d.code_layout = 1;
    }
    if (tc_coarse_supported(nl, h.d)) {
        std::vector<float> tc, norms;
        build_tc_centroids(h.centroids.data(), nl, h.d, tc, norms);
        PG_TRY(dmalloc(&d.cent_tc, tc.size(), acct));
        PG_TRY(dmalloc(&d.cent_norm, norms.size(), acct));
        PG_CUDA(cudaMemcpy(d.cent_tc, tc.data(), tc.size() * 4, cudaMemcpyHostToDevice));
        PG_CUDA(cudaMemcpy(d.cent_norm, norms.data(), norms.size() * 4, cudaMemcpyHostToDevice));
        d.tc_ok = true;
    }
    return PRAG_GPU_OK;
}

int finish_load(std::unique_ptr<prag_gpu_index>& ix, HostIndex& h, int device, prag_gpu_index** out) {
    DeviceGuard g(device);
    ix->device = device;
    ix->ntotal_global = h.ntotal_global ? h.ntotal_global : h.ids.size();
    int rc = upload(ix.get(), h);
    if (rc != PRAG_GPU_OK) {
        free_device_index(ix->dev);
        return rc;
    }
    *out = ix.release();
    return PRAG_GPU_OK;
}

// ------------------------------------------------------------ workspace
Workspace* acquire_ws(prag_gpu_index* ix, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(ix->mu);
    for (Workspace* w : ix->pool) {
        if (w->busy) continue;
        if (w->last_stream == s || cudaEventQuery(w->done) == cudaSuccess) {
            w->busy = true;
            return w;
        }
    }
    cudaGetLastError();
    auto* w = new Workspace();
    w->device = ix->device;
    cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&w->host_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&w->xev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&w->xev2, cudaEventDisableTiming);
    for (auto& e : w->ev) cudaEventCreate(&e);
    if (cudaMalloc(&w->sync, 64) == cudaSuccess) cudaMemset(w->sync, 0, 64);
    else w->sync = nullptr;
    cudaGetLastError();
    w->busy = true;
    ix->pool.push_back(w);
    return w;
}

void release_ws(prag_gpu_index* ix, Workspace* w, cudaStream_t s) {
    cudaEventRecord(w->done, s);
    w->last_stream = s;
    std::lock_guard<std::mutex> lk(ix->mu);
    w->busy = false;
}

int ws_reserve(Workspace* w, size_t bytes, cudaStream_t s) {
    if (w->buf_bytes >= bytes) return PRAG_GPU_OK;
    if (w->buf) {
        PG_CUDA(cudaStreamSynchronize(s));
        cudaFree(w->buf);
        w->buf = nullptr;
        w->buf_bytes = 0;
    }
    size_t b = std::max(bytes, w->buf_bytes * 2);
    if (cudaMalloc(&w->buf, b) != cudaSuccess) {
        cudaGetLastError();
        PG_CUDA(cudaMalloc(&w->buf, bytes));
        b = bytes;
    }
    w->buf_bytes = b;
    return PRAG_GPU_OK;
}

int ws_reserve_x(Workspace* w, size_t bytes, cudaStream_t s) {
    if (w->xbuf_bytes >= bytes) return PRAG_GPU_OK;
    if (w->xbuf) {
        PG_CUDA(cudaStreamSynchronize(s));
        cudaFree(w->xbuf);
        w->xbuf = nullptr;
        w->xbuf_bytes = 0;
    }
    PG_CUDA(cudaMalloc(&w->xbuf, bytes));
    w->xbuf_bytes = bytes;
    return PRAG_GPU_OK;
}

void free_ws(Workspace* w) {
    if (!w) return;
    cudaFree(w->buf);
    cudaFree(w->stage);
    cudaFree(w->xbuf);
    cudaFree(w->win_stat);
    cudaFree(w->sync);
    if (w->host) cudaFreeHost(w->host);
    if (w->done) cudaEventDestroy(w->done);
    if (w->host_ev) cudaEventDestroy(w->host_ev);
    if (w->xev) cudaEventDestroy(w->xev);
    if (w->xev2) cudaEventDestroy(w->xev2);
    for (auto& e : w->ev)
        if (e) cudaEventDestroy(e);
    delete w;
}

std::vector<uint64_t> prefix_desc(const std::vector<uint64_t>& sizes) {
    std::vector<uint64_t> sorted(sizes);
    std::sort(sorted.begin(), sorted.end(), std::greater<uint64_t>());
    std::vector<uint64_t> p(sorted.size() + 1, 0);
    for (size_t i = 0; i < sorted.size(); ++i) p[i + 1] = p[i] + sorted[i];
    return p;
}

int ws_reserve_stage(Workspace* w, size_t bytes, cudaStream_t s) {
    if (w->stage_bytes >= bytes) return PRAG_GPU_OK;
    if (w->stage) {
        PG_CUDA(cudaStreamSynchronize(s));
        cudaFree(w->stage);
        w->stage = nullptr;
        w->stage_bytes = 0;
    }
    PG_CUDA(cudaMalloc(&w->stage, bytes));
    w->stage_bytes = bytes;
    return PRAG_GPU_OK;
}

int ws_reserve_host(Workspace* w, size_t bytes) {
    if (w->host_bytes >= bytes) return PRAG_GPU_OK;
    if (w->host_pending) PG_CUDA(cudaEventSynchronize(w->host_ev));
    w->host_pending = false;
    if (w->host) cudaFreeHost(w->host);
    w->host = nullptr;
    size_t b = std::max(bytes, w->host_bytes * 2);
    PG_CUDA(cudaMallocHost(&w->host, b));
    w->host_bytes = b;
    return PRAG_GPU_OK;
}


uint32_t pow2_at_least(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return uint32_t(p);
}

int blocks_per_sm_scan(const prag_gpu_index* ix) {
    const size_t lut = size_t(ix->dev.nsq) * 1024 + ((ix->dev.d + 3) & ~3u) * 4;
    int per = lut <= 200 * 1024 ? int((228 * 1024) / (lut + 1024)) : 4;
    return std::max(1, std::min(per, 8));
}

// K1 + K1b: the first nprobe lists of each query in (distance, list id)
// order. Tensor-core pre-filter + exact window rescoring when the shape
// allows (coarse_tc.cu), else the exact SIMT scan of every centroid.
// Scratch: coarse holds coarse_scratch_floats() (K1's per-slice partial dot
// products, or the exact distances); pkey/ptie nq * pw.
bool use_tc_coarse(const prag_gpu_index* ix, uint32_t nprobe) {
    return ix->dev.tc_ok && ix->coarse_path == 0 && nprobe <= kTcMaxNprobe;
}

size_t coarse_scratch_floats(const prag_gpu_index* ix, uint32_t nq) {
    return size_t(nq) * ix->dev.nlist * (ix->dev.tc_ok ? std::max<uint32_t>(1, tc_slices(ix->dev.d)) : 1);
}

int run_coarse(const prag_gpu_index* ix, const float* dq, uint32_t nq, uint32_t nprobe, float* coarse,
               uint32_t* probe, float* probe_dist, uint32_t* pkey, uint64_t* ptie, cudaStream_t s,
               Workspace* prof_ws) {
    const DeviceIndex& d = ix->dev;
    unsigned long long* win_stat = nullptr;
    if (prof_ws) {  // profiling: event between K1 and K1b, window-size counter
        if (!prof_ws->win_stat) PG_CUDA(cudaMalloc(&prof_ws->win_stat, 8));
        PG_CUDA(cudaMemsetAsync(prof_ws->win_stat, 0, 8, s));
        win_stat = prof_ws->win_stat;
    }
    if (use_tc_coarse(ix, nprobe)) {
        PG_TRY(launch_coarse_tc(d, dq, nq, coarse, s));
        if (prof_ws) cudaEventRecord(prof_ws->ev[1], s);
        return launch_select_window(d, coarse, dq, nq, nprobe, probe, probe_dist, win_stat, s);
    }
    PG_TRY(launch_coarse(d, dq, nq, coarse, s));
    if (prof_ws) cudaEventRecord(prof_ws->ev[1], s);
    return launch_select_probe(d, coarse, nq, nprobe, probe, probe_dist, pkey, ptie, s);
}

// PRAG_GPU_SPLIT_ITEMS (tuning knob, scan_skew.cu launch_lut_images): extra
// work-item capacity when it asks for more split items than the default.
static uint64_t split_items_override() {
    const char* e = getenv("PRAG_GPU_SPLIT_ITEMS");
    return e ? 3ull * uint64_t(std::max(0, atoi(e))) : 0ull;
}

// Fast path (m = 32 / 64, k <= 32): coarse -> top-nprobe -> plan -> LUT
// images -> fused conflict-free scan + warp top-k -> pool select.
int search_pass_skew(prag_gpu_index* ix, Workspace* w, const float* dq, uint32_t nq, uint32_t nprobe, uint32_t k,
                     uint64_t* o_ids, float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s,
                     prag_gpu_timings* tm) {
    const DeviceIndex& d = ix->dev;
    const int sms = search_sms(ix);
    const int grid = sms;  // persistent: one CTA per SM (of the search's SM budget)
    if (w->sync && search1_eligible(d, nq, nprobe, k, sms)) {
        // one query: the whole search in one launch (batch1.cu)
        PG_TRY(ws_reserve(w, search1_scratch_bytes(d, nprobe, grid), s));
        if (tm) cudaEventRecord(w->ev[0], s);
        PG_TRY(launch_search1(d, dq, nprobe, k, o_ids, o_dist, o_count, o_scanned, w->buf, w->sync, grid, s));
        if (tm) {
            cudaEventRecord(w->ev[5], s);
            PG_CUDA(cudaEventSynchronize(w->ev[5]));
            float tot;
            cudaEventElapsedTime(&tot, w->ev[0], w->ev[5]);
            tm->scan_ms += tot;  // one kernel: coarse, tables, scan and merge
            tm->total_ms += tot;
            uint64_t sc = 0;
            PG_CUDA(cudaMemcpy(&sc, o_scanned, 8, cudaMemcpyDeviceToHost));
            tm->scanned_bytes += sc * d.nsq;
        }
        return PRAG_GPU_OK;
    }
    // item size from the worst-case tile count of this shape (host-side, so a
    // given (nq, nprobe) always plans the same way)
    const uint64_t max_tiles_q = (ix->top_prefix[nprobe] + 31) / 32 + nprobe;
    const uint32_t IT = skew_item_tiles(uint64_t(nq) * max_tiles_q, uint32_t(grid));
    // + the tail items the planner may split (kSplit - 1 = 3 extra per split item)
    const uint64_t item_cap = uint64_t(nq) * (nprobe + max_tiles_q / IT + 1) + 1 + split_items_override();
    const uint64_t pool_cap = item_cap * k;  // k entries per work item
    const uint32_t pw_p = pow2_at_least(nprobe);
    const uint32_t pw_f = pow2_at_least(std::max<uint64_t>(1, std::min<uint64_t>(k, pool_cap)));
    const uint64_t img_floats = uint64_t(nq) * nprobe * (skew_lut_bytes(d.nsq) / 4);  // K3 LUT images
    size_t need;
    {
        Carver c{nullptr};
        c.take<float>(coarse_scratch_floats(ix, nq));
        c.take<uint32_t>(size_t(nq) * nprobe);
        c.take<float>(size_t(nq) * nprobe);
        c.take<uint32_t>(size_t(nq) * pw_p);
        c.take<uint64_t>(size_t(nq) * pw_p);
        c.take<uint4>(item_cap);
        c.take<uint32_t>(2);
        c.take<uint32_t>(size_t(nq) + 1);
        c.take<uint32_t>(nq);
        c.take<uint32_t>(size_t(nq) * nprobe);
        c.take<uint32_t>(pool_cap);
        c.take<uint64_t>(pool_cap);
        c.take<uint32_t>(size_t(nq) * pw_f);
        c.take<uint64_t>(size_t(nq) * pw_f);
        c.take<float>(img_floats);
        need = c.off + 1024;
    }
    PG_TRY(ws_reserve(w, need, s));
    Carver c{static_cast<char*>(w->buf)};
    float* coarse = c.take<float>(coarse_scratch_floats(ix, nq));
    uint32_t* probe = c.take<uint32_t>(size_t(nq) * nprobe);
    float* probe_dist = c.take<float>(size_t(nq) * nprobe);
    uint32_t* pkey = c.take<uint32_t>(size_t(nq) * pw_p);
    uint64_t* ptie = c.take<uint64_t>(size_t(nq) * pw_p);
    uint4* items = c.take<uint4>(item_cap);
    uint32_t* ctr = c.take<uint32_t>(2);
    uint32_t* q_item_off = c.take<uint32_t>(size_t(nq) + 1);
    uint32_t* gthr = c.take<uint32_t>(nq);
    uint32_t* pair_off = c.take<uint32_t>(size_t(nq) * nprobe);
    uint32_t* pool_key = c.take<uint32_t>(pool_cap);
    uint64_t* pool_id = c.take<uint64_t>(pool_cap);
    uint32_t* fkey = c.take<uint32_t>(size_t(nq) * pw_f);
    uint64_t* ftie = c.take<uint64_t>(size_t(nq) * pw_f);
    float* images = c.take<float>(img_floats);

    const bool prof = tm != nullptr;
    if (prof) cudaEventRecord(w->ev[0], s);
    PG_TRY(run_coarse(ix, dq, nq, nprobe, coarse, probe, probe_dist, pkey, ptie, s, prof ? w : nullptr));
    if (prof) cudaEventRecord(w->ev[2], s);
    PG_TRY(launch_lut_images(d, dq, probe, nq, nprobe, images, IT, o_scanned, items, ctr, ctr + 1, q_item_off, gthr,
                             pair_off, item_cap, uint32_t(grid), s));
    if (prof) cudaEventRecord(w->ev[3], s);
    PG_TRY(launch_scan_skew(d, items, ctr, ctr + 1, probe, images, nprobe, k, gthr, pool_key, pool_id, grid, s));
    if (prof) cudaEventRecord(w->ev[4], s);
    PG_TRY(launch_select_pool(pool_key, pool_id, d.ids, o_scanned, q_item_off, gthr, nq, k, o_ids, o_dist, o_count, fkey,
                              ftie, pw_f, s));
    if (prof) {
        cudaEventRecord(w->ev[5], s);
        PG_CUDA(cudaEventSynchronize(w->ev[5]));
        float t[5];
        for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], w->ev[i], w->ev[i + 1]);
        float tot;
        cudaEventElapsedTime(&tot, w->ev[0], w->ev[5]);
        tm->coarse_ms += t[0];
        tm->select_ms += t[1];
        tm->plan_ms += t[2];  // plan + LUT images
        tm->scan_ms += t[3];
        tm->final_ms += t[4];
        tm->total_ms += tot;
        std::vector<uint64_t> sc(nq);
        PG_CUDA(cudaMemcpy(sc.data(), o_scanned, nq * 8, cudaMemcpyDeviceToHost));
        for (uint64_t v : sc) tm->scanned_bytes += v * d.nsq;
        uint32_t ni = 0;
        PG_CUDA(cudaMemcpy(&ni, ctr, 4, cudaMemcpyDeviceToHost));
        tm->work_items += ni;
        unsigned long long wsum = 0;
        if (use_tc_coarse(ix, nprobe)) PG_CUDA(cudaMemcpy(&wsum, w->win_stat, 8, cudaMemcpyDeviceToHost));
        tm->coarse_window += wsum;
    }
    return PRAG_GPU_OK;
}

// One pass over nq (<= chunk) device-resident queries. Outputs are device
// pointers. All launches on stream s.
int search_pass(prag_gpu_index* ix, Workspace* w, const float* dq, uint32_t nq, uint32_t nprobe, uint32_t k,
                uint64_t* o_ids, float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s,
                prag_gpu_timings* tm, bool rerank) {
    const DeviceIndex& d = ix->dev;
    if (!rerank && d.code_layout == 1 && k <= 32 && ix->scan_path == 0)
        return search_pass_skew(ix, w, dq, nq, nprobe, k, o_ids, o_dist, o_count, o_scanned, s, tm);
    const uint64_t max_cand_q = ix->top_prefix[nprobe];
    const uint64_t cand_cap = std::max<uint64_t>(1, max_cand_q * nq);
    const uint32_t C = scan_chunk();
    const uint64_t item_cap = uint64_t(nq) * (nprobe + (max_cand_q + C - 1) / C) + 1;
    const uint32_t pw_p = pow2_at_least(nprobe);
    const uint32_t pw_f = pow2_at_least(std::max<uint64_t>(1, std::min<uint64_t>(k, max_cand_q)));
    const int sms = search_sms(ix);
    const int per_sm = blocks_per_sm_scan(ix);
    const int grid = int(std::max<uint64_t>(1, std::min<uint64_t>(item_cap, uint64_t(sms) * per_sm)));
    const size_t lut_bytes = size_t(d.nsq) * 1024 + ((d.d + 3) & ~3u) * 4;
    const bool glut = lut_bytes > 200 * 1024;

    size_t need = 0;
    {
        Carver c{nullptr};
        c.take<float>(coarse_scratch_floats(ix, nq));
        c.take<uint32_t>(size_t(nq) * nprobe);
        c.take<float>(size_t(nq) * nprobe);
        c.take<uint32_t>(size_t(nq) * pw_p);
        c.take<uint64_t>(size_t(nq) * pw_p);
        c.take<uint64_t>(size_t(nq) + 1);
        c.take<uint4>(item_cap);
        c.take<uint32_t>(2);
        c.take<float>(cand_cap);
        c.take<uint32_t>(cand_cap);
        c.take<uint32_t>(size_t(nq) * pw_f);
        c.take<uint64_t>(size_t(nq) * pw_f);
        if (glut) c.take<float>(size_t(grid) * d.nsq * 256);
        need = c.off + 256;
    }
    PG_TRY(ws_reserve(w, need, s));
    Carver c{static_cast<char*>(w->buf)};
    SearchBuffers b{};
    b.queries = dq;
    b.nq = nq;
    b.nprobe = nprobe;
    b.k = k;
    b.out_ids = o_ids;
    b.out_dist = o_dist;
    b.out_count = o_count;
    b.out_scanned = o_scanned;
    b.coarse_dist = c.take<float>(coarse_scratch_floats(ix, nq));
    b.probe = c.take<uint32_t>(size_t(nq) * nprobe);
    b.probe_dist = c.take<float>(size_t(nq) * nprobe);
    uint32_t* pkey = c.take<uint32_t>(size_t(nq) * pw_p);
    uint64_t* ptie = c.take<uint64_t>(size_t(nq) * pw_p);
    b.q_cand_off = c.take<uint64_t>(size_t(nq) + 1);
    b.items = c.take<uint4>(item_cap);
    uint32_t* ctr = c.take<uint32_t>(2);
    b.num_items = ctr;
    b.item_cursor = ctr + 1;
    b.cand_dist = c.take<float>(cand_cap);
    b.cand_entry = c.take<uint32_t>(cand_cap);
    uint32_t* fkey = c.take<uint32_t>(size_t(nq) * pw_f);
    uint64_t* ftie = c.take<uint64_t>(size_t(nq) * pw_f);
    float* gl = glut ? c.take<float>(size_t(grid) * d.nsq * 256) : nullptr;
    b.item_cap = item_cap;
    b.cand_cap = cand_cap;

    const bool prof = tm != nullptr;
    if (prof) cudaEventRecord(w->ev[0], s);
    PG_TRY(run_coarse(ix, dq, nq, nprobe, b.coarse_dist, b.probe, b.probe_dist, pkey, ptie, s, prof ? w : nullptr));
    if (prof) cudaEventRecord(w->ev[2], s);
    PG_TRY(launch_plan(d, b, s));
    if (prof) cudaEventRecord(w->ev[3], s);
    PG_TRY(launch_scan(d, b, s, grid, gl));
    if (rerank) PG_TRY(launch_rerank(d, b, ix->emb, max_cand_q, s));
    if (prof) cudaEventRecord(w->ev[4], s);
    PG_TRY(launch_final(d, b, fkey, ftie, pw_f, s));
    if (prof) {
        cudaEventRecord(w->ev[5], s);
        PG_CUDA(cudaEventSynchronize(w->ev[5]));
        float t[5];
        for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], w->ev[i], w->ev[i + 1]);
        float tot;
        cudaEventElapsedTime(&tot, w->ev[0], w->ev[5]);
        tm->coarse_ms += t[0];
        tm->select_ms += t[1];
        tm->plan_ms += t[2];
        tm->scan_ms += t[3];
        tm->final_ms += t[4];
        tm->total_ms += tot;
        std::vector<uint64_t> sc(nq);
        PG_CUDA(cudaMemcpy(sc.data(), o_scanned, nq * 8, cudaMemcpyDeviceToHost));
        for (uint64_t v : sc) tm->scanned_bytes += v * d.nsq;
        uint32_t ni = 0;
        PG_CUDA(cudaMemcpy(&ni, b.num_items, 4, cudaMemcpyDeviceToHost));
        tm->work_items += ni;
        unsigned long long wsum = 0;
        if (use_tc_coarse(ix, nprobe)) PG_CUDA(cudaMemcpy(&wsum, w->win_stat, 8, cudaMemcpyDeviceToHost));
        tm->coarse_window += wsum;
    }
    return PRAG_GPU_OK;
}

int validate(const prag_gpu_index* ix, uint32_t nprobe, uint32_t k) {
    if (k < 1) {  // annindex.hpp:265
        set_error("search: k must be >= 1");
        return PRAG_GPU_CONFIG;
    }
    if (nprobe < 1 || nprobe > ix->dev.nlist) {  // annindex.hpp:266-268
        set_error("search: nprobe out of [1, nlist]");
        return PRAG_GPU_CONFIG;
    }
    return PRAG_GPU_OK;
}

bool uses_fast_path(const prag_gpu_index* ix, uint32_t k, bool rerank) {
    return !rerank && ix->dev.code_layout == 1 && k <= 32 && ix->scan_path == 0;
}

uint32_t pass_chunk(const prag_gpu_index* ix, uint32_t nq, uint32_t nprobe, uint32_t k, bool rerank) {
    // Bound candidate memory: chunk the batch so a pass holds <= 192M slots.
    const std::vector<uint64_t>& tp = ix->global_top_prefix.empty() ? ix->top_prefix : ix->global_top_prefix;
    const uint64_t max_cand_q = std::max<uint64_t>(1, tp[nprobe]);
    const uint64_t kSlots = 192ull << 20;
    uint32_t chunk = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(nq, kSlots / max_cand_q)));
    if (uses_fast_path(ix, k, rerank)) {
        // fast path: bound the per-pass LUT images (nq * nprobe * m * 2 KiB) to ~1 GiB
        const uint64_t img_q = uint64_t(nprobe) * skew_lut_bytes(ix->dev.nsq);
        chunk = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(nq, (1ull << 30) / img_q)));
    }
    return chunk;
}

// One pass of whatever this handle is: a single index (search_pass), a
// group of shards (group_pass: per-shard passes + the peer-memory merge), or
// a rank of a distributed index (dist_pass: local pass + NCCL all-gather +
// merge). Device queries in, device outputs out, on stream s.
static int any_pass(prag_gpu_index* ix, Workspace* w, const float* dq, uint32_t nq, uint32_t nprobe, uint32_t k,
                    uint64_t* o_ids, float* o_dist, uint32_t* o_count, uint64_t* o_scanned, cudaStream_t s,
                    prag_gpu_timings* tm, bool rerank) {
    if (ix->is_group()) return group_pass(ix, w, dq, nq, nprobe, k, o_ids, o_dist, o_count, o_scanned, s, rerank,
                                          nullptr);
    if (ix->comm) return dist_pass(ix, w, dq, nq, nprobe, k, o_ids, o_dist, o_count, o_scanned, s, tm, rerank);
    return search_pass(ix, w, dq, nq, nprobe, k, o_ids, o_dist, o_count, o_scanned, s, tm, rerank);
}

void free_host_plan(HostPlan* h) {
    if (!h) return;
    if (h->plan) prag_gpu_plan_free(h->plan);
    cudaFree(h->dq);
    cudaFree(h->dout);
    cudaFreeHost(h->hout);
    delete h;
}

// Small host-buffer searches (nq <= kHostPlanMaxNq: GpuRetriever's batch-1
// retrieve) replay a captured plan per (nq, nprobe, k, stream) shape: one H2D
// copy, one graph launch, one D2H copy of the four outputs, instead of the
// chain's kernel launches. Measured (tools/host_path_time.py, config B, wall
// clock per call): batch 1 at nprobe 1 / 16 / 128 48 / 57 / 85 us with the
// plan vs 56 / 57 / 93 us without; nq 16 / 64 slower with the plan (122 vs
// 108, 206 vs 203 us: the graph loses the PDL overlap the direct launches
// keep), so larger batches take the direct path. Up to kHostPlans shapes per
// index are kept (least recently used evicted). Returns -1 when the call
// should take the ordinary path (a larger batch, another call holds the
// shape's plan, profiling, a sharded handle, or PRAG_GPU_HOST_PLANS=0).
constexpr size_t kHostPlans = 8;
constexpr uint32_t kHostPlanMaxNq = 4;

int host_plan_search(prag_gpu_index* ix, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t k,
                     uint64_t* out_ids, float* out_dist, uint32_t* out_count, uint64_t* out_scanned,
                     cudaStream_t s) {
    static const bool enabled = [] {
        const char* e = getenv("PRAG_GPU_HOST_PLANS");
        return !(e && e[0] == '0');
    }();
    if (!enabled || nq > kHostPlanMaxNq || ix->profiling || ix->is_group() || ix->comm ||
        pass_chunk(ix, nq, nprobe, k, false) < nq)
        return -1;
    static std::atomic<uint64_t> clock{0};
    HostPlan* hp = nullptr;
    {
        std::lock_guard<std::mutex> lk(ix->mu);
        for (HostPlan* h : ix->host_plans)
            if (h->nq == nq && h->nprobe == nprobe && h->k == k && h->stream == s) {
                if (h->busy) return -1;
                hp = h;
                break;
            }
        if (hp) hp->busy = true;
    }
    const DeviceIndex& d = ix->dev;
    Carver c{nullptr};
    c.take<uint64_t>(size_t(nq) * k);
    c.take<float>(size_t(nq) * k);
    c.take<uint32_t>(nq);
    c.take<uint64_t>(nq);
    const size_t out_bytes = c.off;
    auto carve = [&](char* base, uint64_t** i, float** dd, uint32_t** cnt, uint64_t** sc) {
        Carver v{base};
        *i = v.take<uint64_t>(size_t(nq) * k);
        *dd = v.take<float>(size_t(nq) * k);
        *cnt = v.take<uint32_t>(nq);
        *sc = v.take<uint64_t>(nq);
    };
    if (!hp) {  // build the shape's plan (an ordinary pass, then its capture)
        auto h = std::make_unique<HostPlan>();
        h->nq = nq, h->nprobe = nprobe, h->k = k, h->stream = s, h->out_bytes = out_bytes;
        struct Guard {
            std::unique_ptr<HostPlan>& h;
            ~Guard() {
                if (h) free_host_plan(h.release());
            }
        } guard{h};
        PG_CUDA(cudaMalloc(&h->dq, size_t(nq) * d.d * 4));
        PG_CUDA(cudaMalloc(&h->dout, out_bytes));
        PG_CUDA(cudaMallocHost(&h->hout, out_bytes));
        PG_CUDA(cudaMemcpyAsync(h->dq, queries, size_t(nq) * d.d * 4, cudaMemcpyHostToDevice, s));
        uint64_t *i, *sc;
        float* dd;
        uint32_t* cnt;
        carve(h->dout, &i, &dd, &cnt, &sc);
        PG_TRY(prag_gpu_plan_create(ix, h->dq, nq, nprobe, k, i, dd, cnt, sc, s, &h->plan));
        h->busy = true;
        HostPlan* evict = nullptr;
        {
            std::lock_guard<std::mutex> lk(ix->mu);
            if (ix->host_plans.size() >= kHostPlans) {
                auto it = std::min_element(ix->host_plans.begin(), ix->host_plans.end(), [](HostPlan* a, HostPlan* b) {
                    return (a->busy ? UINT64_MAX : a->last_use) < (b->busy ? UINT64_MAX : b->last_use);
                });
                if (!(*it)->busy) {
                    evict = *it;
                    ix->host_plans.erase(it);
                }
            }
            hp = h.release();
            ix->host_plans.push_back(hp);
        }
        if (evict) free_host_plan(evict);
    } else {
        PG_CUDA(cudaMemcpyAsync(hp->dq, queries, size_t(nq) * d.d * 4, cudaMemcpyHostToDevice, s));
    }
    struct Release {
        prag_gpu_index* ix;
        HostPlan* hp;
        ~Release() {
            std::lock_guard<std::mutex> lk(ix->mu);
            hp->busy = false;
            hp->last_use = ++clock;
        }
    } rel{ix, hp};
    PG_TRY(prag_gpu_plan_launch(hp->plan, s));
    PG_CUDA(cudaMemcpyAsync(hp->hout, hp->dout, out_bytes, cudaMemcpyDeviceToHost, s));
    PG_CUDA(cudaStreamSynchronize(s));
    uint64_t *hi, *hs;
    float* hd;
    uint32_t* hc;
    carve(hp->hout, &hi, &hd, &hc, &hs);
    std::memcpy(out_ids, hi, size_t(nq) * k * 8);
    std::memcpy(out_dist, hd, size_t(nq) * k * 4);
    std::memcpy(out_count, hc, size_t(nq) * 4);
    if (out_scanned) std::memcpy(out_scanned, hs, size_t(nq) * 8);
    return PRAG_GPU_OK;
}

int do_search(prag_gpu_index* ix, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t k,
              uint64_t* out_ids, float* out_dist, uint32_t* out_count, uint64_t* out_scanned, cudaStream_t s,
              bool rerank, bool all_device) {
    PG_TRY(validate(ix, nprobe, k));
    const bool has_emb = ix->is_group() ? ix->shards[0]->emb != nullptr : ix->emb != nullptr;
    if (rerank && !has_emb) {  // annindex.hpp:269-271
        set_error("search: exact_rerank requires raw embeddings");
        return PRAG_GPU_CONFIG;
    }
    if (nq == 0) return PRAG_GPU_OK;
    if (!queries || !out_ids || !out_dist || !out_count) {
        set_error("search: null query/output pointer");
        return PRAG_GPU_CONFIG;
    }
    DeviceGuard g(ix->device);
    const DeviceIndex& d = ix->dev;
    // (all_device: the caller vouches that every pointer is device memory,
    // which skips five pointer-attribute queries on the launch path)
    const bool q_dev = all_device || is_device_ptr(queries);
    const bool o_dev = all_device || (is_device_ptr(out_ids) && is_device_ptr(out_dist) && is_device_ptr(out_count) &&
                                      (out_scanned == nullptr || is_device_ptr(out_scanned)));
    const uint32_t chunk = pass_chunk(ix, nq, nprobe, k, rerank);
    if (!q_dev && !o_dev && !rerank) {
        const int rc = host_plan_search(ix, queries, nq, nprobe, k, out_ids, out_dist, out_count, out_scanned, s);
        if (rc >= 0) return rc;
    }

    Workspace* w = acquire_ws(ix, s);
    struct Rel {
        prag_gpu_index* ix;
        Workspace* w;
        cudaStream_t s;
        ~Rel() { release_ws(ix, w, s); }
    } rel{ix, w, s};

    // device staging for host queries/outputs (and scanned scratch), kept
    // in the workspace so it follows the same stream-ordered reuse rules
    const size_t qbytes = size_t(chunk) * d.d * 4;
    const size_t obytes = size_t(chunk) * k * 12 + size_t(chunk) * 12 + 1024;
    PG_TRY(ws_reserve_stage(w, qbytes + obytes + 512, s));
    float* dq_stage = static_cast<float*>(w->stage);
    char* do_stage = static_cast<char*>(w->stage) + ((qbytes + 255) & ~size_t(255));
    if (!q_dev || !o_dev) PG_TRY(ws_reserve_host(w, std::max(qbytes, obytes) + 256));
    prag_gpu_timings tm{};
    prag_gpu_timings* tmp = ix->profiling ? &tm : nullptr;
    const bool q_pinned = !q_dev && is_pinned_host(queries);
    for (uint32_t q0 = 0; q0 < nq; q0 += chunk) {
        const uint32_t n = std::min(chunk, nq - q0);
        const float* dq;
        if (q_dev) {
            dq = queries + size_t(q0) * d.d;
        } else {
            const float* src = queries + size_t(q0) * d.d;
            if (q_pinned) {
                PG_CUDA(cudaMemcpyAsync(dq_stage, src, size_t(n) * d.d * 4, cudaMemcpyHostToDevice, s));
            } else {
                if (w->host_pending) PG_CUDA(cudaEventSynchronize(w->host_ev));
                std::memcpy(w->host, src, size_t(n) * d.d * 4);
                PG_CUDA(cudaMemcpyAsync(dq_stage, w->host, size_t(n) * d.d * 4, cudaMemcpyHostToDevice, s));
                PG_CUDA(cudaEventRecord(w->host_ev, s));
                w->host_pending = true;
            }
            dq = dq_stage;
        }
        uint64_t* oi;
        float* od;
        uint32_t* oc;
        uint64_t* os;
        size_t stage_out_bytes = 0;
        if (o_dev) {
            oi = out_ids + size_t(q0) * k;
            od = out_dist + size_t(q0) * k;
            oc = out_count + q0;
            os = out_scanned ? out_scanned + q0 : reinterpret_cast<uint64_t*>(do_stage);
        } else {
            Carver cv{do_stage};
            oi = cv.take<uint64_t>(size_t(n) * k);
            od = cv.take<float>(size_t(n) * k);
            oc = cv.take<uint32_t>(n);
            os = cv.take<uint64_t>(n);
            stage_out_bytes = cv.off;
        }
        PG_TRY(any_pass(ix, w, dq, n, nprobe, k, oi, od, oc, os, s, tmp, rerank));
        if (!o_dev) {
            // device -> pinned -> caller: the four outputs sit in one staged
            // block, so one copy brings them back (same carve offsets)
            char* h = static_cast<char*>(w->host);
            Carver hv{h};
            uint64_t* hi = hv.take<uint64_t>(size_t(n) * k);
            float* hd = hv.take<float>(size_t(n) * k);
            uint32_t* hc = hv.take<uint32_t>(n);
            uint64_t* hs = hv.take<uint64_t>(n);
            PG_CUDA(cudaMemcpyAsync(h, do_stage, stage_out_bytes, cudaMemcpyDeviceToHost, s));
            PG_CUDA(cudaStreamSynchronize(s));
            std::memcpy(out_ids + size_t(q0) * k, hi, size_t(n) * k * 8);
            std::memcpy(out_dist + size_t(q0) * k, hd, size_t(n) * k * 4);
            std::memcpy(out_count + q0, hc, size_t(n) * 4);
            if (out_scanned) std::memcpy(out_scanned + q0, hs, size_t(n) * 8);
        }
    }
    if (tmp) {
        std::lock_guard<std::mutex> lk(ix->mu);
        ix->last = tm;
    }
    return PRAG_GPU_OK;
}


}  // namespace pg

namespace pg {

int build_synthetic(uint32_t nlist, uint32_t d, uint32_t nsq, uint64_t ntotal, uint64_t seed, double sigma,
                    const float* centroids, const float* codewords, int rank, int world, int device,
                    prag_gpu_index** out) {
    if (!out || !centroids || !codewords) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) {
        set_error("invalid shard arguments");
        return PRAG_GPU_CONFIG;
    }
    if ((nsq != 32 && nsq != 64) || d % nsq != 0 || d / nsq > 16 || d % 4 != 0 || nlist == 0) {
        set_error("synthetic index: needs m in {32, 64}, d % m == 0, d / m <= 16, d % 4 == 0, nlist >= 1");
        return PRAG_GPU_CONFIG;
    }
    PG_TRY(require_device(device));
    DeviceGuard g(device);
    auto ix = std::make_unique<prag_gpu_index>();
    ix->device = device;
    ix->ntotal_global = ntotal;
    DeviceIndex& dv = ix->dev;
    dv.nlist = nlist;
    dv.d = d;
    dv.nsq = nsq;
    dv.sub_dim = d / nsq;
    dv.plain_codes = false;
    std::vector<uint64_t> sizes;  // the whole index's lists
    synth_list_sizes(nlist, ntotal, seed, sigma, sizes);
    // shard: the entry ranges prag_gpu_plan_shard_ranges gives `rank` (whole
    // lists, or a stripe of a large one); every entry keeps its global
    // list-major position g (chunk id g, codes from g)
    std::vector<uint64_t> rsz(sizes), rbeg(nlist, 0);
    if (world > 1) {
        std::vector<uint64_t> rend(nlist);
        plan_shard_ranges(sizes.data(), nlist, uint32_t(world), uint32_t(rank), rbeg.data(), rend.data());
        for (uint32_t l = 0; l < nlist; ++l) rsz[l] = rend[l] - rbeg[l];
    }
    ix->shard_rank = rank;
    ix->shard_world = world;
    ix->global_top_prefix = prefix_desc(sizes);
    std::vector<uint64_t> gbase(size_t(nlist) + 1, 0), poff(size_t(nlist) + 1, 0), soff(size_t(nlist) + 1, 0);
    std::vector<uint32_t> len(nlist);
    uint32_t maxlen = 0;
    uint64_t resident = 0;
    for (uint32_t l = 0; l < nlist; ++l) {
        if (sizes[l] >= (1ull << 32)) {
            set_error("synthetic index: list exceeds 2^32 entries");
            return PRAG_GPU_CONFIG;
        }
        len[l] = uint32_t(rsz[l]);
        maxlen = std::max(maxlen, len[l]);
        resident += rsz[l];
        gbase[l + 1] = gbase[l] + sizes[l];
        poff[l + 1] = poff[l] + (rsz[l] + kListPad - 1) / kListPad * kListPad;
        soff[l + 1] = soff[l] + (rsz[l] ? (rsz[l] + 31) / 32 + 1 : 0);
    }
    if (poff[nlist] >= (1ull << 32)) {
        set_error("more than 2^32 resident entries on one device; shard the index");
        return PRAG_GPU_CONFIG;
    }
    dv.ntotal = resident;
    dv.npadded = poff[nlist];
    dv.max_list_len = maxlen;
    ix->host_list_len = rsz;
    ix->top_prefix = prefix_desc(rsz);
    uint64_t* acct = &ix->device_bytes;
    auto fail = [&](int rc) {
        free_device_index(dv);
        return rc;
    };
    int rc = PRAG_GPU_OK;
    uint64_t* dloff = nullptr;  // [2][nlist + 1]: global entry base, resident length
    const size_t cw = size_t(nsq) * 256 * (d / nsq);
    std::vector<float> t(size_t(nlist) * d);
    if ((rc = dmalloc(&dv.centroids, size_t(nlist) * d, acct)) ||
        (rc = dmalloc(&dv.centroids4, size_t(nlist) * d, acct)) || (rc = dmalloc(&dv.codewordsT, cw, acct)) ||
        (rc = dmalloc(&dv.codewords, cw, acct)) || (rc = dmalloc(&dv.list_off, size_t(nlist) + 1, acct)) ||
        (rc = dmalloc(&dv.list_len, nlist, acct)) || (rc = dmalloc(&dv.skew_off, size_t(nlist) + 1, acct)) ||
        (rc = dmalloc(&dv.ids, dv.npadded, acct)) || (rc = dmalloc(&dv.skew_codes, soff[nlist] * 32 * nsq, acct)) ||
        (rc = dmalloc(&dloff, 2 * (size_t(nlist) + 1), nullptr)))
        return fail(rc);
    for (uint32_t c = 0; c < nlist; ++c)
        for (uint32_t j = 0; j < d; ++j) t[(size_t(j / 4) * nlist + c) * 4 + (j % 4)] = centroids[size_t(c) * d + j];
    std::vector<float> wt(cw);
    const uint32_t sub = d / nsq;
    for (uint32_t sq = 0; sq < nsq; ++sq)
        for (uint32_t c = 0; c < 256; ++c)
            for (uint32_t j = 0; j < sub; ++j) wt[(size_t(sq) * sub + j) * 256 + c] = codewords[(size_t(sq) * 256 + c) * sub + j];
    cudaError_t e = cudaSuccess;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
        if (e == cudaSuccess) e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
    };
    cp(dv.centroids, centroids, size_t(nlist) * d * 4);
    cp(dv.centroids4, t.data(), t.size() * 4);
    cp(dv.codewordsT, wt.data(), cw * 4);
    cp(dv.codewords, codewords, cw * 4);
    cp(dv.list_off, poff.data(), poff.size() * 8);
    cp(dv.list_len, len.data(), len.size() * 4);
    cp(dv.skew_off, soff.data(), soff.size() * 8);
    std::vector<uint64_t> ebase(gbase);  // global position of each list's first resident entry
    for (uint32_t l = 0; l < nlist; ++l) ebase[l] += rbeg[l];
    cp(dloff, ebase.data(), ebase.size() * 8);
    cp(dloff + nlist + 1, rsz.data(), size_t(nlist) * 8);
    if (e != cudaSuccess) {
        cudaFree(dloff);
        set_error(std::string("CUDA error (synthetic index upload): ") + cudaGetErrorString(e));
        return fail(PRAG_GPU_CUDA);
    }
    rc = launch_synth_codes(nsq, dloff, dloff + nlist + 1, dv.skew_off, nlist, seed, dv.skew_codes, soff[nlist], dv.ids,
                            dv.list_off, dv.npadded);
    cudaFree(dloff);
    if (rc) return fail(rc);
    dv.code_layout = 1;
    if (tc_coarse_supported(nlist, d)) {
        std::vector<float> tc, norms;
        build_tc_centroids(centroids, nlist, d, tc, norms);
        if ((rc = dmalloc(&dv.cent_tc, tc.size(), acct)) || (rc = dmalloc(&dv.cent_norm, norms.size(), acct)))
            return fail(rc);
        cp(dv.cent_tc, tc.data(), tc.size() * 4);
        cp(dv.cent_norm, norms.data(), norms.size() * 4);
        if (e != cudaSuccess) {
            set_error(std::string("CUDA error (synthetic index upload): ") + cudaGetErrorString(e));
            return fail(PRAG_GPU_CUDA);
        }
        dv.tc_ok = true;
    }
    *out = ix.release();
    return PRAG_GPU_OK;
}


}  // namespace pg

using namespace pg;

extern "C" {

const char* prag_gpu_last_error(void) { return g_error.c_str(); }
int prag_gpu_version(void) { return 1; }

int prag_gpu_device_count(void) {
    PG_API_BEGIN
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
    PG_API_END
}

int prag_gpu_index_load(const char* path, int device, prag_gpu_index** out) {
    PG_API_BEGIN
    if (!out || !path) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    *out = nullptr;
    PG_TRY(require_device(device));
    HostIndex h;
    PG_TRY(read_pragix01(path, h, nullptr));
    auto ix = std::make_unique<prag_gpu_index>();
    return finish_load(ix, h, device, out);
    PG_API_END
}

int prag_gpu_index_load_shard(const char* path, int device, int rank, int world, prag_gpu_index** out) {
    PG_API_BEGIN
    if (!out || !path || world < 1 || rank < 0 || rank >= world) {
        set_error("invalid shard arguments");
        return PRAG_GPU_CONFIG;
    }
    *out = nullptr;
    PG_TRY(require_device(device));
    std::vector<uint64_t> sizes;
    PG_TRY(read_pragix01_list_sizes(path, sizes));
    KeepRanges keep;
    keep.begin.resize(sizes.size());
    keep.end.resize(sizes.size());
    plan_shard_ranges(sizes.data(), uint32_t(sizes.size()), uint32_t(world), uint32_t(rank), keep.begin.data(),
                      keep.end.data());
    HostIndex h;
    PG_TRY(read_pragix01(path, h, &keep));
    auto ix = std::make_unique<prag_gpu_index>();
    ix->shard_rank = rank;
    ix->shard_world = world;
    ix->global_top_prefix = prefix_desc(sizes);
    return finish_load(ix, h, device, out);
    PG_API_END
}

int prag_gpu_index_synthetic(uint32_t nlist, uint32_t d, uint32_t nsq, uint64_t ntotal, uint64_t seed, double sigma,
                             const float* centroids, const float* codewords, int device, prag_gpu_index** out) {
    PG_API_BEGIN
    return build_synthetic(nlist, d, nsq, ntotal, seed, sigma, centroids, codewords, 0, 1, device, out);
    PG_API_END
}

int prag_gpu_index_synthetic_shard(uint32_t nlist, uint32_t d, uint32_t nsq, uint64_t ntotal, uint64_t seed,
                                   double sigma, const float* centroids, const float* codewords, int rank,
                                   int world, int device, prag_gpu_index** out) {
    PG_API_BEGIN
    return build_synthetic(nlist, d, nsq, ntotal, seed, sigma, centroids, codewords, rank, world, device, out);
    PG_API_END
}

int prag_gpu_index_from_host(uint32_t nlist, uint32_t d, uint32_t nsq, const float* centroids,
                             const float* codewords, const uint64_t* list_off, const uint64_t* ids,
                             const uint8_t* codes, int device, prag_gpu_index** out) {
    PG_API_BEGIN
    if (!out) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    *out = nullptr;
    if (nsq == 0 || d % nsq != 0) {
        set_error("invalid n_subquantizers");
        return PRAG_GPU_CONFIG;
    }
    PG_TRY(require_device(device));
    HostIndex h;
    h.nlist = nlist;
    h.d = d;
    h.nsq = nsq;
    h.sub_dim = d / nsq;
    h.centroids.assign(centroids, centroids + size_t(nlist) * d);
    h.codewords.assign(codewords, codewords + size_t(nsq) * 256 * (d / nsq));
    h.list_off.assign(list_off, list_off + nlist + 1);
    const uint64_t n = list_off[nlist];
    for (uint32_t l = 0; l < nlist; ++l)
        if (list_off[l + 1] < list_off[l]) {
            set_error("list_off must be non-decreasing");
            return PRAG_GPU_CONFIG;
        }
    h.ids.assign(ids, ids + n);
    h.codes.assign(codes, codes + n * nsq);
    h.ntotal_global = n;
    auto ix = std::make_unique<prag_gpu_index>();
    return finish_load(ix, h, device, out);
    PG_API_END
}

void prag_gpu_index_free(prag_gpu_index* ix) {
    if (!ix) return;
    if (ix->is_group()) {
        free_group(ix);
        delete ix;
        return;
    }
    {
        DeviceGuard g(ix->device);
        cudaDeviceSynchronize();
        for (HostPlan* h : ix->host_plans) free_host_plan(h);
        ix->host_plans.clear();
        for (Workspace* w : ix->pool) free_ws(w);
        free_device_index(ix->dev);
        cudaFree(ix->emb);
    }
    delete ix;
}

int prag_gpu_index_describe(const prag_gpu_index* ix, prag_gpu_index_desc* o) {
    PG_API_BEGIN
    if (!ix || !o) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    std::memset(o, 0, sizeof *o);
    o->nlist = ix->dev.nlist;
    o->d = ix->dev.d;
    o->nsq = ix->dev.nsq;
    o->sub_dim = ix->dev.sub_dim;
    o->ntotal = ix->dev.ntotal;
    o->ntotal_global = ix->ntotal_global;
    o->max_list_len = ix->dev.max_list_len;
    o->device = ix->device;
    o->shard_rank = ix->shard_rank;
    o->shard_world = ix->shard_world;
    o->device_bytes = ix->device_bytes;
    o->code_layout = ix->dev.code_layout;
    if (ix->is_group()) {  // the whole index, over shards.size() shards
        o->shard_world = int32_t(ix->shards.size());
        o->device_bytes = 0;
        for (const prag_gpu_index* sh : ix->shards) o->device_bytes += sh->device_bytes;
    }
    return PRAG_GPU_OK;
    PG_API_END
}

uint32_t prag_gpu_index_nlist(const prag_gpu_index* ix) { return ix ? ix->dev.nlist : 0; }

int prag_gpu_index_list_sizes(const prag_gpu_index* ix, uint64_t* out) {
    PG_API_BEGIN
    if (!ix || !out) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    std::copy(ix->host_list_len.begin(), ix->host_list_len.end(), out);
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_search(prag_gpu_index* ix, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t k,
                    uint64_t* out_ids, float* out_dist, uint32_t* out_count, uint64_t* out_scanned,
                    void* stream) {
    PG_API_BEGIN
    if (!ix) {
        set_error("null index");
        return PRAG_GPU_CONFIG;
    }
    return do_search(ix, queries, nq, nprobe, k, out_ids, out_dist, out_count, out_scanned,
                     static_cast<cudaStream_t>(stream));
    PG_API_END
}

int prag_gpu_index_store(const prag_gpu_index* ix, const char* path) {
    PG_API_BEGIN
    if (!ix || !path) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    const DeviceIndex& d = ix->dev;
    if (ix->shard_world > 1 || ix->is_group()) {
        set_error("store: a shard holds only part of the lists; store the full index");
        return PRAG_GPU_CONFIG;
    }
    DeviceGuard g(ix->device);
    const uint32_t nl = d.nlist, sub = d.d / d.nsq;
    std::vector<float> cent(size_t(nl) * d.d), words(size_t(d.nsq) * 256 * sub);
    std::vector<uint64_t> off(size_t(nl) + 1), ids(d.npadded);
    std::vector<uint32_t> len(nl);
    std::vector<uint8_t> codes(d.npadded * d.nsq);
    if (d.codes) {
        PG_CUDA(cudaMemcpy(codes.data(), d.codes, codes.size(), cudaMemcpyDeviceToHost));
    } else {  // only the lane-skewed tiles are resident: undo the skew (scan_skew.cu)
        std::vector<uint64_t> soff(size_t(nl) + 1), off2(size_t(nl) + 1);
        std::vector<uint32_t> len2(nl);
        PG_CUDA(cudaMemcpy(soff.data(), d.skew_off, soff.size() * 8, cudaMemcpyDeviceToHost));
        PG_CUDA(cudaMemcpy(off2.data(), d.list_off, off2.size() * 8, cudaMemcpyDeviceToHost));
        PG_CUDA(cudaMemcpy(len2.data(), d.list_len, len2.size() * 4, cudaMemcpyDeviceToHost));
        const uint32_t m = d.nsq;
        std::vector<uint8_t> tiles;
        for (uint32_t l = 0; l < nl; ++l) {
            const uint64_t nt = soff[l + 1] - soff[l];
            if (!nt) continue;
            tiles.resize(nt * 32 * m);
            PG_CUDA(cudaMemcpy(tiles.data(), d.skew_codes + soff[l] * 32 * m, tiles.size(), cudaMemcpyDeviceToHost));
            for (uint32_t e = 0; e < len2[l]; ++e) {
                const uint32_t t = e & 31u;
                for (uint32_t b = 0; b < m; ++b) {
                    uint32_t tile = e >> 5, s = b + t;
                    bool tail = false;
                    if (s >= m) {
                        s -= m;
                        ++tile;
                        tail = true;
                    }
                    const uint8_t v = tiles[size_t(tile) * 32 * m + (s >> 4) * 512 + t * 16 + (s & 15u)];
                    codes[(off2[l] + e) * m + b] = (tail && m == 64) ? uint8_t(v - 1) : v;
                }
            }
        }
    }
    PG_CUDA(cudaMemcpy(cent.data(), d.centroids, cent.size() * 4, cudaMemcpyDeviceToHost));
    PG_CUDA(cudaMemcpy(words.data(), d.codewords, words.size() * 4, cudaMemcpyDeviceToHost));
    PG_CUDA(cudaMemcpy(off.data(), d.list_off, off.size() * 8, cudaMemcpyDeviceToHost));
    PG_CUDA(cudaMemcpy(len.data(), d.list_len, len.size() * 4, cudaMemcpyDeviceToHost));
    PG_CUDA(cudaMemcpy(ids.data(), d.ids, ids.size() * 8, cudaMemcpyDeviceToHost));
    // annindex.hpp:335-359 layout, written to a temporary then renamed
    const std::string tmp = std::string(path) + ".tmp";
    FILE* f = fopen(tmp.c_str(), "wb");
    if (!f) {
        set_error(std::string("cannot open for writing: ") + path);
        return PRAG_GPU_FORMAT;
    }
    const uint32_t hdr[4] = {1u, nl, d.d, d.nsq};
    bool ok = fwrite("PRAGIX01", 1, 8, f) == 8 && fwrite(hdr, 4, 4, f) == 4 &&
              fwrite(cent.data(), 4, cent.size(), f) == cent.size() &&
              fwrite(words.data(), 4, words.size(), f) == words.size();
    std::vector<uint8_t> rec;
    for (uint32_t l = 0; ok && l < nl; ++l) {
        const uint64_t n = len[l];
        ok = fwrite(&n, 8, 1, f) == 1;
        rec.resize(size_t(n) * (8 + d.nsq));
        for (uint64_t e = 0; e < n; ++e) {
            std::memcpy(&rec[e * (8 + d.nsq)], &ids[off[l] + e], 8);
            std::memcpy(&rec[e * (8 + d.nsq) + 8], &codes[(off[l] + e) * d.nsq], d.nsq);
        }
        ok = ok && (n == 0 || fwrite(rec.data(), 1, rec.size(), f) == rec.size());
    }
    ok = (fclose(f) == 0) && ok;
    if (!ok || std::rename(tmp.c_str(), path) != 0) {
        std::remove(tmp.c_str());
        set_error(std::string("write failed: ") + path);
        return PRAG_GPU_FORMAT;
    }
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_search_device(prag_gpu_index* ix, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t k,
                           uint64_t* out_ids, float* out_dist, uint32_t* out_count, uint64_t* out_scanned,
                           void* stream) {
    PG_API_BEGIN
    if (!ix) {
        set_error("null index");
        return PRAG_GPU_CONFIG;
    }
    return do_search(ix, queries, nq, nprobe, k, out_ids, out_dist, out_count, out_scanned,
                     static_cast<cudaStream_t>(stream), false, true);
    PG_API_END
}

}  // extern "C"


extern "C" {

int prag_gpu_plan_create(prag_gpu_index* ix, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t k,
                         uint64_t* out_ids, float* out_dist, uint32_t* out_count, uint64_t* out_scanned,
                         void* stream, prag_gpu_plan** out) {
    PG_API_BEGIN
    if (!ix || !out || !queries || !out_ids || !out_dist || !out_count || !out_scanned || nq == 0) {
        set_error("plan: null argument or empty batch");
        return PRAG_GPU_CONFIG;
    }
    *out = nullptr;
    PG_TRY(validate(ix, nprobe, k));
    if (!(is_device_ptr(queries) && is_device_ptr(out_ids) && is_device_ptr(out_dist) && is_device_ptr(out_count) &&
          is_device_ptr(out_scanned))) {
        set_error("plan: queries and outputs must be device memory");
        return PRAG_GPU_CONFIG;
    }
    if (pass_chunk(ix, nq, nprobe, k, false) < nq) {
        set_error("plan: batch too large for one pass (split it)");
        return PRAG_GPU_CONFIG;
    }
    DeviceGuard g(ix->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto plan = std::make_unique<prag_gpu_plan>();
    plan->ix = ix;
    if (ix->is_group()) {  // per-shard graphs on their own devices + the root merge
        PG_TRY(group_plan_create(ix, queries, nq, nprobe, k, out_ids, out_dist, out_count, out_scanned, s,
                                 &plan->group));
        *out = plan.release();
        return PRAG_GPU_OK;
    }
    plan->w = new Workspace();
    plan->w->device = ix->device;
    PG_CUDA(cudaEventCreateWithFlags(&plan->w->done, cudaEventDisableTiming));
    struct Cleanup {
        prag_gpu_plan* p;
        ~Cleanup() {
            if (!p) return;
            if (p->exec) cudaGraphExecDestroy(p->exec);
            if (p->graph) cudaGraphDestroy(p->graph);
            free_ws(p->w);
        }
    } cleanup{plan.get()};
    // one ordinary pass sizes the plan's own workspace, then the same pass is
    // captured (no allocation or host synchronisation inside it). On a
    // distributed shard both passes are collective (every rank creates the
    // plan) and the capture holds the NCCL all-gather.
    PG_TRY(any_pass(ix, plan->w, queries, nq, nprobe, k, out_ids, out_dist, out_count, out_scanned, s, nullptr,
                    false));
    PG_CUDA(cudaStreamSynchronize(s));
    // capture on a private stream: the caller's may be the legacy default
    // stream, which cannot be captured (the graph launches on any stream)
    cudaStream_t cap = nullptr;
    PG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    struct CapStream {
        cudaStream_t s;
        ~CapStream() { cudaStreamDestroy(s); }
    } cap_guard{cap};
    PG_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    const int rc = any_pass(ix, plan->w, queries, nq, nprobe, k, out_ids, out_dist, out_count, out_scanned, cap,
                            nullptr, false);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cap, &graph);
    if (rc != PRAG_GPU_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    PG_CUDA(ce);
    plan->graph = graph;
    PG_CUDA(cudaGraphInstantiate(&plan->exec, graph, 0));
    cleanup.p = nullptr;
    *out = plan.release();
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_plan_launch(prag_gpu_plan* plan, void* stream) {
    PG_API_BEGIN
    if (plan && plan->group) return group_plan_launch(plan->ix, plan->group, static_cast<cudaStream_t>(stream));
    if (!plan || !plan->exec) {
        set_error("plan: null plan");
        return PRAG_GPU_CONFIG;
    }
    PG_CUDA(cudaGraphLaunch(plan->exec, static_cast<cudaStream_t>(stream)));
    return PRAG_GPU_OK;
    PG_API_END
}

void prag_gpu_plan_free(prag_gpu_plan* plan) {
    if (!plan) return;
    if (plan->group) {
        group_plan_free(plan->ix, plan->group);
        delete plan;
        return;
    }
    DeviceGuard g(plan->ix->device);
    cudaDeviceSynchronize();
    if (plan->exec) cudaGraphExecDestroy(plan->exec);
    if (plan->graph) cudaGraphDestroy(plan->graph);
    free_ws(plan->w);
    delete plan;
}

int prag_gpu_search_rerank(prag_gpu_index* ix, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t k,
                           uint64_t* out_ids, float* out_dist, uint32_t* out_count, uint64_t* out_scanned,
                           void* stream) {
    PG_API_BEGIN
    if (!ix) {
        set_error("null index");
        return PRAG_GPU_CONFIG;
    }
    return do_search(ix, queries, nq, nprobe, k, out_ids, out_dist, out_count, out_scanned,
                     static_cast<cudaStream_t>(stream), true);
    PG_API_END
}

int prag_gpu_index_set_embeddings(prag_gpu_index* ix, const float* emb, uint64_t n) {
    PG_API_BEGIN
    if (!ix || (!emb && n)) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    if (ix->is_group()) {  // every shard reranks its own candidates
        for (prag_gpu_index* sh : ix->shards) PG_TRY(prag_gpu_index_set_embeddings(sh, emb, n));
        return PRAG_GPU_OK;
    }
    DeviceGuard g(ix->device);
    PG_CUDA(cudaDeviceSynchronize());
    cudaFree(ix->emb);
    ix->emb = nullptr;
    ix->emb_n = 0;
    if (n == 0) return PRAG_GPU_OK;
    // every resident chunk id must have a row (annindex.hpp:310 indexes by chunk id)
    uint64_t max_id = 0;
    PG_TRY(max_chunk_id(ix->dev.ids, ix->dev.npadded, &max_id));
    if (ix->dev.ntotal && max_id >= n) {
        set_error("set_embeddings: chunk id " + std::to_string(max_id) + " has no embedding row (n = " +
                  std::to_string(n) + ")");
        return PRAG_GPU_CONFIG;
    }
    const size_t bytes = size_t(n) * ix->dev.d * 4;
    float* e = nullptr;
    PG_CUDA(cudaMalloc(&e, bytes));
    const cudaError_t err = cudaMemcpy(e, emb, bytes, cudaMemcpyDefault);
    if (err != cudaSuccess) {
        cudaFree(e);
        set_error(std::string("CUDA error (set_embeddings): ") + cudaGetErrorString(err));
        return PRAG_GPU_CUDA;
    }
    ix->emb = e;
    ix->emb_n = n;
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_brute_force(const float* vectors, uint64_t n, uint32_t d, const float* queries, uint32_t nq,
                         uint32_t k, int device, uint64_t* out_ids, float* out_dist, uint32_t* out_count) {
    PG_API_BEGIN
    if (k < 1) {  // annindex.hpp:246
        set_error("brute_force_search: k must be >= 1");
        return PRAG_GPU_CONFIG;
    }
    if (nq == 0) return PRAG_GPU_OK;
    if ((!vectors && n) || !queries || !out_ids || !out_dist || !out_count || d == 0) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    if (n > 0xffffffffull) {
        set_error("brute_force_search: the device path takes n < 2^32 rows");
        return PRAG_GPU_CONFIG;
    }
    PG_TRY(require_device(device));
    DeviceGuard g(device);
    struct Bufs {
        void* p[8] = {};
        ~Bufs() {
            for (void* x : p) cudaFree(x);
        }
    } b;
    const float* emb = vectors;
    if (!is_device_ptr(vectors) && n) {
        PG_CUDA(cudaMalloc(&b.p[0], size_t(n) * d * 4));
        PG_CUDA(cudaMemcpy(b.p[0], vectors, size_t(n) * d * 4, cudaMemcpyHostToDevice));
        emb = static_cast<float*>(b.p[0]);
    }
    const uint32_t pw = pow2_at_least(k);
    // queries per pass: the [chunk][n] distance scratch stays <= 1 GiB
    const uint32_t chunk = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(nq, (1ull << 28) / std::max<uint64_t>(n, 1))));
    PG_CUDA(cudaMalloc(&b.p[1], std::max<size_t>(size_t(chunk) * n * 4, 4)));
    PG_CUDA(cudaMalloc(&b.p[2], size_t(chunk) * pw * 4));
    PG_CUDA(cudaMalloc(&b.p[3], size_t(chunk) * pw * 8));
    PG_CUDA(cudaMalloc(&b.p[4], size_t(chunk) * d * 4));
    PG_CUDA(cudaMalloc(&b.p[5], size_t(chunk) * k * 8));
    PG_CUDA(cudaMalloc(&b.p[6], size_t(chunk) * k * 4));
    PG_CUDA(cudaMalloc(&b.p[7], size_t(chunk) * 4));
    for (uint32_t q0 = 0; q0 < nq; q0 += chunk) {
        const uint32_t m = std::min(chunk, nq - q0);
        PG_CUDA(cudaMemcpy(b.p[4], queries + size_t(q0) * d, size_t(m) * d * 4, cudaMemcpyDefault));
        PG_TRY(launch_brute_force(emb, n, d, static_cast<float*>(b.p[4]), m, k, static_cast<float*>(b.p[1]),
                                  static_cast<uint32_t*>(b.p[2]), static_cast<uint64_t*>(b.p[3]), pw,
                                  static_cast<uint64_t*>(b.p[5]), static_cast<float*>(b.p[6]),
                                  static_cast<uint32_t*>(b.p[7]), nullptr));
        PG_CUDA(cudaMemcpy(out_ids + size_t(q0) * k, b.p[5], size_t(m) * k * 8, cudaMemcpyDefault));
        PG_CUDA(cudaMemcpy(out_dist + size_t(q0) * k, b.p[6], size_t(m) * k * 4, cudaMemcpyDefault));
        PG_CUDA(cudaMemcpy(out_count + q0, b.p[7], size_t(m) * 4, cudaMemcpyDefault));
    }
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_probe(prag_gpu_index* ix, const float* queries, uint32_t nq, uint32_t nprobe, uint32_t* out_lists,
                   float* out_dist, void* stream) {
    PG_API_BEGIN
    if (!ix) {
        set_error("null index");
        return PRAG_GPU_CONFIG;
    }
    PG_TRY(validate(ix, nprobe, 1));
    if (nq == 0) return PRAG_GPU_OK;
    if (ix->is_group()) ix = ix->shards[0];  // centroids are replicated: every shard has the probe order
    DeviceGuard g(ix->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const DeviceIndex& d = ix->dev;
    const uint32_t pw = pow2_at_least(nprobe);
    Workspace* w = acquire_ws(ix, s);
    struct Rel {
        prag_gpu_index* ix;
        Workspace* w;
        cudaStream_t s;
        ~Rel() { release_ws(ix, w, s); }
    } rel{ix, w, s};
    size_t need;
    {
        Carver c{nullptr};
        c.take<float>(size_t(nq) * d.d);
        c.take<float>(coarse_scratch_floats(ix, nq));
        c.take<uint32_t>(size_t(nq) * nprobe);
        c.take<float>(size_t(nq) * nprobe);
        c.take<uint32_t>(size_t(nq) * pw);
        c.take<uint64_t>(size_t(nq) * pw);
        need = c.off + 256;
    }
    PG_TRY(ws_reserve(w, need, s));
    Carver c{static_cast<char*>(w->buf)};
    float* dq = c.take<float>(size_t(nq) * d.d);
    float* coarse = c.take<float>(coarse_scratch_floats(ix, nq));
    uint32_t* pl = c.take<uint32_t>(size_t(nq) * nprobe);
    float* pd = c.take<float>(size_t(nq) * nprobe);
    uint32_t* pk = c.take<uint32_t>(size_t(nq) * pw);
    uint64_t* pt = c.take<uint64_t>(size_t(nq) * pw);
    PG_CUDA(cudaMemcpyAsync(dq, queries, size_t(nq) * d.d * 4, cudaMemcpyDefault, s));
    PG_TRY(run_coarse(ix, dq, nq, nprobe, coarse, pl, pd, pk, pt, s));
    PG_CUDA(cudaMemcpyAsync(out_lists, pl, size_t(nq) * nprobe * 4, cudaMemcpyDefault, s));
    if (out_dist) PG_CUDA(cudaMemcpyAsync(out_dist, pd, size_t(nq) * nprobe * 4, cudaMemcpyDefault, s));
    PG_CUDA(cudaStreamSynchronize(s));
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_plan_shards(const uint64_t* sizes, uint32_t nlist, uint32_t world, uint32_t* owner) {
    PG_API_BEGIN
    if ((!sizes || !owner) && nlist) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    if (world < 1) {
        set_error("world must be >= 1");
        return PRAG_GPU_CONFIG;
    }
    plan_shards_lpt(sizes, nlist, world, owner);
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_plan_shard_ranges(const uint64_t* sizes, uint32_t nlist, uint32_t world, uint32_t rank,
                               uint64_t* out_begin, uint64_t* out_end) {
    PG_API_BEGIN
    if ((!sizes || !out_begin || !out_end) && nlist) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    if (world < 1 || rank >= world) {
        set_error("world must be >= 1 and rank < world");
        return PRAG_GPU_CONFIG;
    }
    plan_shard_ranges(sizes, nlist, world, rank, out_begin, out_end);
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_merge_topk(const uint64_t* ids, const float* dist, const uint32_t* count, const uint64_t* scanned,
                        uint32_t nparts, uint32_t nq, uint32_t kin, uint32_t k, uint64_t* out_ids,
                        float* out_dist, uint32_t* out_count, uint64_t* out_scanned, int device, void* stream) {
    PG_API_BEGIN
    if (k < 1) {
        set_error("merge: k must be >= 1");
        return PRAG_GPU_CONFIG;
    }
    if (nq == 0 || nparts == 0) return PRAG_GPU_OK;
    PG_TRY(require_device(device));
    DeviceGuard g(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t cap = size_t(nparts) * kin;
    const uint32_t pw = pow2_at_least(std::max<uint64_t>(1, std::min<uint64_t>(k, cap)));
    Carver c{nullptr};
    c.take<uint64_t>(cap * nq);
    c.take<float>(cap * nq);
    c.take<uint32_t>(size_t(nparts) * nq);
    c.take<uint64_t>(size_t(nparts) * nq);
    c.take<uint64_t>(size_t(nq) * k);
    c.take<float>(size_t(nq) * k);
    c.take<uint32_t>(nq);
    c.take<uint64_t>(nq);
    c.take<uint32_t>(cap * nq);
    c.take<uint64_t>(cap * nq);
    c.take<uint32_t>(size_t(nq) * pw);
    c.take<uint64_t>(size_t(nq) * pw);
    void* buf = nullptr;
    PG_CUDA(cudaMallocAsync(&buf, c.off + 256, s));
    Carver v{static_cast<char*>(buf)};
    uint64_t* di = v.take<uint64_t>(cap * nq);
    float* dd = v.take<float>(cap * nq);
    uint32_t* dc = v.take<uint32_t>(size_t(nparts) * nq);
    uint64_t* ds = v.take<uint64_t>(size_t(nparts) * nq);
    uint64_t* oi = v.take<uint64_t>(size_t(nq) * k);
    float* od = v.take<float>(size_t(nq) * k);
    uint32_t* oc = v.take<uint32_t>(nq);
    uint64_t* os = v.take<uint64_t>(nq);
    uint32_t* ck = v.take<uint32_t>(cap * nq);
    uint64_t* ct = v.take<uint64_t>(cap * nq);
    uint32_t* gk = v.take<uint32_t>(size_t(nq) * pw);
    uint64_t* gt = v.take<uint64_t>(size_t(nq) * pw);
    PG_CUDA(cudaMemcpyAsync(di, ids, cap * nq * 8, cudaMemcpyDefault, s));
    PG_CUDA(cudaMemcpyAsync(dd, dist, cap * nq * 4, cudaMemcpyDefault, s));
    PG_CUDA(cudaMemcpyAsync(dc, count, size_t(nparts) * nq * 4, cudaMemcpyDefault, s));
    if (scanned) PG_CUDA(cudaMemcpyAsync(ds, scanned, size_t(nparts) * nq * 8, cudaMemcpyDefault, s));
    PG_TRY(launch_merge(di, dd, dc, scanned ? ds : nullptr, nparts, nq, kin, k, oi, od, oc, os, ck, ct, gk, gt, pw,
                        s));
    PG_CUDA(cudaMemcpyAsync(out_ids, oi, size_t(nq) * k * 8, cudaMemcpyDefault, s));
    PG_CUDA(cudaMemcpyAsync(out_dist, od, size_t(nq) * k * 4, cudaMemcpyDefault, s));
    PG_CUDA(cudaMemcpyAsync(out_count, oc, size_t(nq) * 4, cudaMemcpyDefault, s));
    if (out_scanned) PG_CUDA(cudaMemcpyAsync(out_scanned, os, size_t(nq) * 8, cudaMemcpyDefault, s));
    PG_CUDA(cudaFreeAsync(buf, s));
    if (!(is_device_ptr(out_ids) && is_device_ptr(out_dist) && is_device_ptr(out_count)))
        PG_CUDA(cudaStreamSynchronize(s));
    return PRAG_GPU_OK;
    PG_API_END
}

// ---------------------------------------------------- performance model
static void fit_model(const std::vector<double>& xs, const std::vector<double>& ys, prag_gpu_perf_model* m) {
    // perfmodel.hpp:53-79 least squares + :109-116 clamping
    const size_t n = xs.size();
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    for (size_t i = 0; i < n; ++i) {
        sx += xs[i];
        sy += ys[i];
        sxx += xs[i] * xs[i];
        sxy += xs[i] * ys[i];
    }
    const double denom = n * sxx - sx * sx;
    double slope = 0.0, icpt;
    if (denom == 0.0) {
        icpt = sy / n;
    } else {
        slope = (n * sxy - sx * sy) / denom;
        icpt = (sy - slope * sx) / n;
    }
    double mar = 0.0;
    for (size_t i = 0; i < n; ++i) mar = std::max(mar, std::abs(ys[i] - (slope * xs[i] + icpt)));
    m->slope_s = slope;
    m->intercept_s = icpt;
    m->fit_residual_s = mar;
    m->clamped = 0;
    if (m->slope_s < 0.0) {
        m->slope_s = 0.0;
        m->clamped = 1;
    }
    if (m->intercept_s < 0.0) {
        m->intercept_s = 0.0;
        m->clamped = 1;
    }
}

static double median_of(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

static int calibrate_core(const std::function<int(uint32_t, double*)>& measure, const uint32_t* grid_in,
                          uint32_t grid_len, int repeats, int warmups, prag_gpu_perf_model* out,
                          double* out_lat) {
    if (!out || (!grid_in && grid_len)) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    std::vector<uint32_t> grid(grid_in, grid_in + grid_len);
    std::sort(grid.begin(), grid.end());
    grid.erase(std::unique(grid.begin(), grid.end()), grid.end());
    if (grid.size() < 2) {  // perfmodel.hpp:98
        set_error("calibrate_retrieval: need >= 2 distinct nprobe values");
        return PRAG_GPU_CONFIG;
    }
    if (repeats < 3) {  // perfmodel.hpp:99
        set_error("calibrate_retrieval: repeats must be >= 3");
        return PRAG_GPU_CONFIG;
    }
    std::vector<double> xs, ys;
    for (uint32_t np : grid) {
        double t;
        for (int i = 0; i < warmups; ++i) PG_TRY(measure(np, &t));
        std::vector<double> runs;
        for (int r = 0; r < repeats; ++r) {
            PG_TRY(measure(np, &t));
            runs.push_back(t);
        }
        xs.push_back(double(np));
        ys.push_back(median_of(runs));
    }
    fit_model(xs, ys, out);
    if (out_lat) std::copy(ys.begin(), ys.end(), out_lat);
    return PRAG_GPU_OK;
}

int prag_gpu_calibrate_retrieval(prag_gpu_index* ix, const float* queries, uint32_t nq, uint32_t k,
                                 const uint32_t* grid, uint32_t grid_len, int repeats, int warmups,
                                 prag_gpu_perf_model* out, double* out_lat) {
    PG_API_BEGIN
    if (!ix || !queries || nq == 0) {
        set_error("calibrate: need an index and >= 1 query");
        return PRAG_GPU_CONFIG;
    }
    std::vector<uint64_t> ids(size_t(nq) * k);
    std::vector<float> dist(size_t(nq) * k);
    std::vector<uint32_t> cnt(nq);
    // The drop-in contract: host queries in, host results out, wall clock
    // around the whole call (perfmodel_main.cpp:57-63 Stopwatch protocol).
    auto measure = [&](uint32_t np, double* t) -> int {
        auto t0 = std::chrono::steady_clock::now();
        PG_TRY(prag_gpu_search(ix, queries, nq, np, k, ids.data(), dist.data(), cnt.data(), nullptr, nullptr));
        *t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return PRAG_GPU_OK;
    };
    for (uint32_t i = 0; i < grid_len; ++i)
        if (grid[i] < 1 || grid[i] > ix->dev.nlist) {
            set_error("search: nprobe out of [1, nlist]");
            return PRAG_GPU_CONFIG;
        }
    return calibrate_core(measure, grid, grid_len, repeats, warmups, out, out_lat);
    PG_API_END
}

int prag_gpu_calibrate_with(prag_gpu_measure_fn fn, void* ctx, const uint32_t* grid, uint32_t grid_len,
                            int repeats, int warmups, prag_gpu_perf_model* out) {
    PG_API_BEGIN
    if (!fn) {
        set_error("null measure function");
        return PRAG_GPU_CONFIG;
    }
    auto measure = [&](uint32_t np, double* t) -> int {
        *t = fn(np, ctx);
        return PRAG_GPU_OK;
    };
    return calibrate_core(measure, grid, grid_len, repeats, warmups, out, nullptr);
    PG_API_END
}

uint32_t prag_gpu_select_nprobe(const prag_gpu_perf_model* m, double budget_s, uint32_t nlist, double margin) {
    // perfmodel.hpp:148-157
    if (budget_s <= 0.0) return 1;
    const double limit = budget_s * (1.0 - margin);
    if (m->slope_s * 1 + m->intercept_s > limit) return 1;
    if (m->slope_s <= 0.0) return nlist;
    const double max_n = (limit - m->intercept_s) / m->slope_s;
    if (max_n >= double(nlist)) return nlist;
    return uint32_t(std::max(1.0, std::floor(max_n + 1e-9)));
}

int prag_gpu_set_sm_budget(prag_gpu_index* ix, int sms) {
    PG_API_BEGIN
    if (!ix || sms < 0) {
        set_error("sm budget must be >= 0 (0: every SM)");
        return PRAG_GPU_CONFIG;
    }
    ix->sm_budget = sms;
    for (prag_gpu_index* sh : ix->shards) sh->sm_budget = sms;
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_set_scan_path(prag_gpu_index* ix, int path) {
    PG_API_BEGIN
    if (!ix || path < 0 || path > 1) {
        set_error("scan path must be 0 (auto) or 1 (generic)");
        return PRAG_GPU_CONFIG;
    }
    ix->scan_path = path;
    for (prag_gpu_index* sh : ix->shards) sh->scan_path = path;
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_set_coarse_path(prag_gpu_index* ix, int path) {
    PG_API_BEGIN
    if (!ix || path < 0 || path > 1) {
        set_error("coarse path must be 0 (auto) or 1 (exact SIMT)");
        return PRAG_GPU_CONFIG;
    }
    ix->coarse_path = path;
    for (prag_gpu_index* sh : ix->shards) sh->coarse_path = path;
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_set_profiling(prag_gpu_index* ix, int enabled) {
    PG_API_BEGIN
    if (!ix) {
        set_error("null index");
        return PRAG_GPU_CONFIG;
    }
    ix->profiling = enabled != 0;
    for (prag_gpu_index* sh : ix->shards) sh->profiling = enabled != 0;
    return PRAG_GPU_OK;
    PG_API_END
}

int prag_gpu_last_timings(const prag_gpu_index* ix, prag_gpu_timings* out) {
    PG_API_BEGIN
    if (!ix || !out) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    if (ix->is_group()) ix = ix->shards[0];  // the root shard's passes
    std::lock_guard<std::mutex> lk(const_cast<prag_gpu_index*>(ix)->mu);
    *out = ix->last;
    return PRAG_GPU_OK;
    PG_API_END
}

}  // extern "C"

#ifdef PRAG_CHAIN_TRACE
// Debug build only: op 0 zeroes the chain trace (allocating it on first use),
// op 1 copies its pg::kChainWords values to `out` (see internal.h).
extern "C" int prag_gpu_debug_chain_trace(int op, unsigned long long* out) {
    static unsigned long long* buf = nullptr;
    if (!buf) {
        if (cudaMalloc(&buf, pg::kChainWords * 8) != cudaSuccess) return 3;
        pg::ct_bind_coarse(buf);
        pg::ct_bind_skew(buf);
        pg::ct_bind_kernels(buf);
    }
    if (op == 0) return cudaMemset(buf, 0, pg::kChainWords * 8) == cudaSuccess ? 0 : 3;
    return cudaMemcpy(out, buf, pg::kChainWords * 8, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 3;
}
#endif
