// batch1.cu -- the whole search of ONE query in a single launch.
//
// The pipeline's retrieval call is one query at a time (pipeline.hpp:228:
// `search(..., {nprobe, k, false})` per chunk, k = 2 by default,
// pipeline.hpp:58). The five-kernel chain K1..K4 is latency-bound at that
// shape (a handful of dependent global round trips per kernel), so batch 1
// runs as one persistent grid, one CTA per SM, with two grid barriers:
//
//  1. coarse quantizer (annindex.hpp:277-281): every CTA folds the exact
//     squared_l2(q, c) (common.hpp:73-80, sequential, FMA-free) for a slice of
//     the centroids and publishes its slice's top-nprobe keys
//     (distance bits << 32 | list id: the reference's (distance, list) order);
//     -- grid barrier --
//  2. every CTA selects the global top-nprobe from the per-CTA lists (the
//     nprobe-th smallest list head bounds it; the <= nprobe^2 keys below that
//     bound are bitonic-sorted in SMEM), so all CTAs hold the probe list;
//  3. ADC tables (annindex.hpp:285-299): the CTAs split the nprobe x 256 code
//     rows; a warp computes one row (lane = subquantizer, the reference's
//     per-entry fold) and writes it straight into the conflict-free image
//     layout K3 gathers from (scan_skew.cu SkewSmem), one image per probed
//     list in global memory;
//     -- grid barrier --
//  4. list scan (annindex.hpp:300-305): the probed lists' tiles are cut into
//     one contiguous range per CTA; per list segment the CTA bulk-copies that
//     list's image into SMEM (two buffers: the next segment's copy overlaps
//     this one's scan) and its warps fold their tile ranges exactly as K3 does,
//     keeping an exact warp top-k by (distance, chunk_id) (annindex.hpp:54-60);
//     the CTA's warp lists are merged into the CTA's top-k;
//  5. the last CTA to finish (a ticket counter) merges the CTAs' lists into
//     the final top-k and writes ids, distances, count and scanned_vectors.
//
// Results are bit-identical to the chain (and to the reference): every add
// is the reference's, in the reference's order. Barrier and ticket counters
// live in a per-workspace buffer; they return to their start state at the
// end of every launch, so a captured plan can replay the launch.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.h"
#include "skew_common.cuh"

namespace pg {
namespace {

using namespace skew;

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kMaxProbe = 64;     // nprobe^2 <= kSortCap keys below the head bound
constexpr uint32_t kSortCap = 4096;
constexpr uint32_t kFinalCap = 1024;   // k^2 candidates below the final head bound (k <= 32)
constexpr uint32_t kMaxD = 1024;
constexpr uint32_t kMaxGrid = 256;
constexpr uint32_t kMinWarpTiles = 2;  // a warp re-reads one tail tile per range

template <int M>
struct B1Smem {
    static constexpr uint32_t kGuard = M == 64 ? 128u : 0u;
    static constexpr uint32_t kImg = 65536;
    static constexpr uint32_t kImgStride = kGuard + kImg;
    static constexpr uint32_t kImgSpan = kImgStride + kImg;
    // misc: query, sort keys (phase 5 reuses them), list heads, probe info,
    // image barriers, warp lists
    static constexpr uint32_t kMisc = kMaxD * 4 + kSortCap * 8 + kMaxGrid * 8 + 4 * 4 * (kMaxProbe + 1) + 2 * 8 +
                                      kWarps * 64 * 4;
    static constexpr uint32_t bytes = 225 * 1024;  // (+ static shared memory) within the 227 KiB opt-in
    static_assert((kGuard + kMisc - 16) + kImgSpan + kMisc <= bytes, "batch-1 SMEM exceeds its budget");
};

struct B1Args {
    const float* centroids;    // [nlist][d]
    const float4* centroids4;  // [d/4][nlist][4]
    const float* codewords;    // [nsq][256][sub]
    const uint32_t* list_len;
    const uint64_t* list_off;
    const uint64_t* skew_off;
    const uint8_t* skew_codes;
    const uint64_t* ids;
    uint32_t nlist, d, sub;
    const float* query;
    uint32_t nprobe, k;
    uint64_t* o_ids;
    float* o_dist;
    uint32_t* o_count;
    uint64_t* o_scanned;
    uint64_t* coarse;          // [G][nprobe]
    unsigned char* images;     // [nprobe][kImgStride]
    uint4* caux;               // [G][nprobe] per coarse key: {list_len, list_off, skew_off lo, skew_off hi}
    uint32_t* cand_key;        // [G][32]
    uint64_t* cand_id;         // [G][32]
    unsigned* sync;            // [0] barrier arrivals (2 G per launch), [2] finish ticket
};

// Grid-wide barrier (all CTAs co-resident: cooperative launch): one
// monotone arrival counter per launch, barrier n waits for n * G arrivals
// (one atomic and an acquire-poll, no generation round trip). The CTA that
// takes the last finish ticket -- after every CTA has passed both barriers --
// returns the counter to 0 for the next launch.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(count, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// In-SMEM bitonic sort of n (power of two) 64-bit keys, ascending.
__device__ void bitonic64(uint64_t* a, uint32_t n) {
    for (uint32_t size = 2; size <= n; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < n / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t x = a[lo], y = a[hi];
                if ((x > y) == up) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
            __syncthreads();
        }
    }
}

// The same on (distance bits, chunk id) pairs: (distance, chunk_id) order.
__device__ void bitonic_pairs(uint32_t* key, uint64_t* id, uint32_t n) {
    for (uint32_t size = 2; size <= n; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < n / 2; i += blockDim.x) {
                const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint32_t kx = key[lo], ky = key[hi];
                const uint64_t ix = id[lo], iy = id[hi];
                const bool gt = kx > ky || (kx == ky && ix > iy);
                if (gt == up) {
                    key[lo] = ky;
                    key[hi] = kx;
                    id[lo] = iy;
                    id[hi] = ix;
                }
            }
            __syncthreads();
        }
    }
}

#ifdef PRAG_B1_TRACE
// Debug build only (make EXTRA=-DPRAG_B1_TRACE): globaltimer at the phase
// boundaries, per CTA; read back with prag_gpu_debug_b1_trace.
__device__ unsigned long long g_b1_trace[256 * 16];
#define B1_MARK(i)                                                                           \
    do {                                                                                     \
        if (threadIdx.x == 0) {                                                              \
            unsigned long long t_;                                                           \
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                            \
            g_b1_trace[blockIdx.x * 16 + (i)] = t_;                                          \
        }                                                                                    \
    } while (0)
#else
#define B1_MARK(i) \
    do {           \
    } while (0)
#endif

__device__ __forceinline__ uint32_t pow2_ceil(uint32_t x) { return x <= 1 ? 1u : 1u << (32 - __clz(x - 1)); }

template <int M>
__global__ void __launch_bounds__(kThreads, 1) search1_kernel(const B1Args a) {
    using L = B1Smem<M>;
    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, G = gridDim.x, cta = blockIdx.x;
    const uint32_t base = smem_u32(smem);
    const uint32_t img_off = ((base + L::kGuard + 0xffffu) & ~0xffffu) - base;  // image 0, 64 KiB-aligned
    const uint32_t misc_off = img_off >= L::kGuard + L::kMisc ? 0u : img_off + L::kImgSpan;
    unsigned char* misc = smem + misc_off;
    float* q_s = reinterpret_cast<float*>(misc);
    uint64_t* skey = reinterpret_cast<uint64_t*>(misc + kMaxD * 4);  // [kSortCap]
    uint32_t* skey32 = reinterpret_cast<uint32_t*>(skey);            // phase 5: [kFinalCap] distance bits
    uint64_t* sid = skey + kFinalCap / 2;                            // phase 5: [kFinalCap] chunk ids
    uint64_t* heads = skey + kSortCap;                               // [kMaxGrid]
    uint32_t* probe = reinterpret_cast<uint32_t*>(heads + kMaxGrid);  // [kMaxProbe]
    uint32_t* plen = probe + kMaxProbe;                              // [kMaxProbe]
    uint32_t* toff = plen + kMaxProbe;                               // [kMaxProbe + 1] entry-tile prefix
    uint32_t* scal = toff + kMaxProbe + 1;                           // scalars (> 4)
    uint64_t* bars = reinterpret_cast<uint64_t*>(probe + 4 * (kMaxProbe + 1));
    uint32_t* stash = reinterpret_cast<uint32_t*>(bars + 2);         // [kWarps][64]
    const uint32_t nlist = a.nlist, d = a.d, nprobe = a.nprobe, k = a.k;

    if (tid == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    B1_MARK(0);
    // ---------------------------------------------------------- 1. coarse
    // The slice's centroids are staged [d/4][chunk] float4 in the (not yet
    // used) image region with coalesced loads, one memory round trip per
    // chunk; then thread = centroid folds its row from SMEM (LDS.128,
    // conflict-free), the reference's sequential FMA-free fold.
    const uint32_t per = (nlist + G - 1) / G;
    const uint32_t c0 = cta * per;
    const uint32_t cn = c0 < nlist ? min(per, nlist - c0) : 0u;
    // the list metadata the later phases need travels with the coarse keys
    // (loaded here, in the same round trip as the query and the slice)
    uint4 my_aux = make_uint4(0, 0, 0, 0);
    if (tid < cn) {
        const uint32_t c = c0 + tid;
        const uint64_t so = a.skew_off[c];
        my_aux = make_uint4(a.list_len[c], uint32_t(a.list_off[c]), uint32_t(so), uint32_t(so >> 32));
    }
    for (uint32_t i = tid; i < d; i += kThreads) q_s[i] = a.query[i];
    {
        float4* stg = reinterpret_cast<float4*>(smem + img_off - L::kGuard);
        const uint32_t d4 = d / 4, chunk = min(uint32_t(kThreads), (L::kImgSpan / 16) / d4);
        for (uint32_t cb = 0; cb < cn || cb == 0; cb += chunk) {
            const uint32_t nc = cn > cb ? min(chunk, cn - cb) : 0u;
            for (uint32_t i = tid; i < d4 * nc; i += kThreads) {
                const uint32_t j4 = i / nc, c = i - j4 * nc;
                stg[i] = __ldg(a.centroids4 + size_t(j4) * nlist + c0 + cb + c);
            }
            __syncthreads();
            if (tid < nc) {
                float acc = 0.0f;
                for (uint32_t j4 = 0; j4 < d4; ++j4) {
                    const float4 x = stg[j4 * nc + tid];
                    const float* qq = q_s + 4 * j4;
                    const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float df = __fsub_rn(qq[e], xs[e]);
                        acc = __fadd_rn(acc, __fmul_rn(df, df));
                    }
                }
                skey[cb + tid] = (uint64_t(__float_as_uint(acc)) << 32) | (c0 + cb + tid);
            }
            __syncthreads();
        }
    }
    __syncthreads();
    if (tid < cn) {  // rank within the slice (keys are unique)
        const uint64_t me = skey[tid];
        uint32_t r = 0;
        for (uint32_t i = 0; i < cn; ++i) r += skey[i] < me;
        if (r < nprobe) {
            a.coarse[size_t(cta) * nprobe + r] = me;
            a.caux[size_t(cta) * nprobe + r] = my_aux;
        }
    }
    for (uint32_t r = cn + tid; r < nprobe; r += kThreads) a.coarse[size_t(cta) * nprobe + r] = ~0ull;
    B1_MARK(1);
    grid_barrier(a.sync, G);
    B1_MARK(2);

    // ---------------------------------------------- 2. global top-nprobe
    // U = the nprobe-th smallest list head: the global top-nprobe keys are
    // all <= U, and only the nprobe lists whose head is <= U hold such keys
    // (at most nprobe each).
    __shared__ uint64_t s_u;
    __shared__ uint32_t s_n;
    if (tid == 0) {
        s_u = ~0ull;
        s_n = 0;
    }
    // one pass: every key (and its list metadata) of every CTA's list into
    // registers; the heads go to SMEM for the bound (other CTAs wrote these:
    // read through L2)
    constexpr uint32_t kKpt = (kMaxGrid * kMaxProbe + kThreads - 1) / kThreads;  // keys per thread at most
    const uint32_t nkeys = G * nprobe;
    uint64_t kreg[kKpt];
    uint32_t kidx[kKpt];
#pragma unroll
    for (uint32_t u = 0; u < kKpt; ++u) {
        const uint32_t i = tid + u * kThreads;
        kidx[u] = i;
        kreg[u] = i < nkeys ? __ldcg(a.coarse + i) : ~0ull;
    }
    __syncthreads();  // s_u / s_n initialised
#pragma unroll
    for (uint32_t u = 0; u < kKpt; ++u)
        if (kidx[u] < nkeys && kidx[u] % nprobe == 0) heads[kidx[u] / nprobe] = kreg[u];
    __syncthreads();
    for (uint32_t b = tid; b < G; b += kThreads) {
        const uint64_t h = heads[b];
        uint32_t r = 0;
        for (uint32_t i = 0; i < G; ++i) r += heads[i] < h;
        if (r == nprobe - 1) s_u = h;
    }
    __syncthreads();
    const uint64_t U = s_u;
    uint32_t* sidx = reinterpret_cast<uint32_t*>(smem + img_off - L::kGuard);  // [kSortCap] key -> its slot
#pragma unroll
    for (uint32_t u = 0; u < kKpt; ++u) {
        const uint64_t x = kreg[u];
        if (x <= U && x != ~0ull) {
            const uint32_t pos = atomicAdd(&s_n, 1u);
            if (pos < kSortCap) {
                skey[pos] = x;
                sidx[pos] = kidx[u];
            }
        }
    }
    __syncthreads();
    const uint32_t nsel = min(s_n, kSortCap);
    const uint32_t npad = pow2_ceil(nsel);
    // keys are unique: after sorting, the slot of key x is found by a scan of
    // the unsorted copy (nsel is ~nprobe + a few)
    uint64_t* sunsorted = reinterpret_cast<uint64_t*>(sidx + kSortCap);
    for (uint32_t i = tid; i < nsel; i += kThreads) sunsorted[i] = skey[i];
    for (uint32_t i = nsel + tid; i < npad; i += kThreads) skey[i] = ~0ull;
    __syncthreads();
    bitonic64(skey, npad);
    uint4 paux = make_uint4(0, 0, 0, 0);
    if (tid < nprobe) {
        const uint64_t me = skey[tid];
        uint32_t slot = 0;
        for (uint32_t i = 0; i < nsel; ++i)
            if (sunsorted[i] == me) slot = sidx[i];
        paux = __ldcg(a.caux + slot);
        probe[tid] = uint32_t(me);
        plen[tid] = paux.x;
    }
    uint32_t* plo = reinterpret_cast<uint32_t*>(stash);  // [kMaxProbe] list_off (stash is free until the scan)
    uint64_t* pso = reinterpret_cast<uint64_t*>(plo + kMaxProbe);  // [kMaxProbe] skew_off
    if (tid < nprobe) {
        plo[tid] = paux.y;
        pso[tid] = uint64_t(paux.z) | (uint64_t(paux.w) << 32);
    }
    __syncthreads();
    if (warp == 0) {  // entry-tile prefix over the probed lists, scanned_vectors
        uint32_t carry = 0;
        unsigned long long sc = 0;
        for (uint32_t p0 = 0; p0 < nprobe; p0 += 32) {
            const uint32_t p = p0 + lane;
            const uint32_t t = p < nprobe ? (plen[p] + kTileEntries - 1) / kTileEntries : 0u;
            sc += p < nprobe ? plen[p] : 0u;
            uint32_t incl = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= uint32_t(o)) incl += v;
            }
            if (p < nprobe) toff[p] = carry + incl - t;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        for (int o = 16; o; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
        if (lane == 0) {
            toff[nprobe] = carry;
            scal[0] = uint32_t(sc);
            scal[1] = uint32_t(sc >> 32);
        }
    }
    __syncthreads();
    const uint32_t TT = toff[nprobe];
    const uint32_t tper = max((TT + G - 1) / G, 1u);
    const uint32_t g0 = min(cta * tper, TT), g1 = min(g0 + tper, TT);
    // request this CTA's code tiles into L2 now; they land during the tables
    // (lane 0 of warp w takes the w-th probed list overlapping the range)
    {
        uint32_t seen = 0;
        for (uint32_t p = 0; p < nprobe && g0 < g1; ++p) {
            const uint32_t lo = max(g0, toff[p]), hi = min(g1, toff[p + 1]);
            if (lo >= hi) continue;
            if (warp == seen % kWarps && lane == 0) {
                const unsigned char* src = a.skew_codes + (pso[p] + (lo - toff[p])) * (32ull * M);
                prefetch_l2(src, (hi - lo + 1) * 32u * M);
            }
            ++seen;
        }
    }

    B1_MARK(3);
    // ------------------------------------------------ 3. ADC table images
    // rows (probe p, code) split over the CTAs in contiguous chunks; the
    // residuals q - c_list of the chunk's probes are staged in SMEM (stride
    // sub + 1: conflict-free per subquantizer); a warp computes a row: lane s
    // holds subquantizer s (and s + 32 for m = 64), its codeword loaded whole
    {
        const uint32_t rows = nprobe * 256u, rper = (rows + G - 1) / G;
        const uint32_t r0 = cta * rper, r1 = min(rows, r0 + rper);
        const uint32_t sub = a.sub, rs = sub + 1;
        float* res = reinterpret_cast<float*>(smem + img_off - L::kGuard);  // [probe in chunk][m][sub + 1]
        const uint32_t pbeg = r0 >> 8, pcnt = r0 < r1 ? ((r1 - 1) >> 8) - pbeg + 1 : 0u;
        for (uint32_t i = tid; i < pcnt * d; i += kThreads) {
            const uint32_t pl = i / d, j = i - pl * d;
            const uint32_t list = probe[pbeg + pl];
            res[pl * M * rs + (j / sub) * rs + (j % sub)] = __fsub_rn(q_s[j], __ldg(a.centroids + size_t(list) * d + j));
        }
        __syncthreads();
        for (uint32_t r = r0 + warp; r < r1; r += kWarps) {
            const uint32_t p = r >> 8, code = r & 255u;
            if (plen[p] == 0) continue;
            float* img = reinterpret_cast<float*>(a.images + size_t(p) * L::kImgStride + L::kGuard);
#pragma unroll
            for (int h = 0; h < M / 32; ++h) {
                const uint32_t sq = lane + 32u * h;
                const float* cw = a.codewords + (size_t(sq) * 256 + code) * sub;
                const float* rr = res + (p - pbeg) * M * rs + sq * rs;
                float w[16];
                if (M == 32 && sub == 12) {  // 48-byte codewords: three 16-byte loads up front
                    const float4* c4 = reinterpret_cast<const float4*>(cw);
#pragma unroll
                    for (int u = 0; u < 3; ++u) {
                        const float4 v = __ldg(c4 + u);
                        w[4 * u] = v.x, w[4 * u + 1] = v.y, w[4 * u + 2] = v.z, w[4 * u + 3] = v.w;
                    }
                } else if (M == 64 && sub == 6) {  // 24-byte codewords: three 8-byte loads
                    const float2* c2 = reinterpret_cast<const float2*>(cw);
#pragma unroll
                    for (int u = 0; u < 3; ++u) {
                        const float2 v = __ldg(c2 + u);
                        w[2 * u] = v.x, w[2 * u + 1] = v.y;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (uint32_t(j) < sub) w[j] = __ldg(cw + j);
                }
                float acc = 0.0f;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (uint32_t(j) < sub) {
                        const float df = __fsub_rn(rr[j], w[j]);  // residual - codeword (annindex.hpp:292-297)
                        acc = __fadd_rn(acc, __fmul_rn(df, df));
                    }
                }
                float* row = img + code * 64;
                if (M == 32) {
                    row[sq] = acc;
                    row[sq + 32] = acc;
                } else {
                    row[sq] = acc;
                    if (code == 255 && h == 1) img[int(sq) - 64] = acc;  // guard: row 255's upper half below the image
                }
            }
        }
    }
    // the images are read by other CTAs' bulk copies (the async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    B1_MARK(4);
    grid_barrier(a.sync, 2 * G);
    B1_MARK(5);

    // ------------------------------------------------------------- 4. scan
    float mk[32], nk[32];
#pragma unroll
    for (int s = 0; s < 32; ++s) {
        mk[s] = (uint32_t(s) >= lane) ? 1.0f : 0.0f;
        nk[s] = (uint32_t(s) >= lane) ? 0.0f : 1.0f;
    }
    const uint32_t bt = (31u - lane) * 4u | ((base + img_off) & 0xffff0000u);
    WarpTopK t{0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
    // segments: the probed lists overlapping [g0, g1), in probe order
    uint32_t seg_p[2] = {0, 0};
    uint32_t nseg = 0, next_p = 0;
    auto next_segment = [&](uint32_t& p_out) -> bool {
        while (next_p < nprobe) {
            const uint32_t p = next_p++;
            if (max(g0, toff[p]) < min(g1, toff[p + 1])) {
                p_out = p;
                return true;
            }
        }
        return false;
    };
    auto issue_image = [&](uint32_t b, uint32_t p) {
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bars + b, L::kImgStride);
            bulk_g2s(smem + img_off + b * L::kImgStride - L::kGuard, a.images + size_t(p) * L::kImgStride,
                     L::kImgStride, bars + b);
        }
    };
    {
        uint32_t p;
        if (g0 < g1 && next_segment(p)) {
            seg_p[0] = p;
            issue_image(0, p);
            ++nseg;
            if (next_segment(p)) {
                seg_p[1] = p;
                issue_image(1, p);
                ++nseg;
            }
        }
    }
    uint32_t phase[2] = {0, 0};
    for (uint32_t si = 0; si < nseg; ++si) {
        const uint32_t b = si & 1u, p = seg_p[b];
        const uint32_t lo = max(g0, toff[p]) - toff[p], hi = min(g1, toff[p + 1]) - toff[p];  // entry tiles
        // warp ranges over [lo, hi): >= kMinWarpTiles tiles each; the first two
        // code tiles are requested before waiting for the segment's image
        const uint32_t ntile = hi - lo;
        const uint32_t nw = min(uint32_t(kWarps), (ntile + kMinWarpTiles - 1) / kMinWarpTiles);
        const uint32_t wper = (ntile + nw - 1) / nw;
        const uint32_t wa = lo + warp * wper, we = min(hi, wa + wper);
        const bool active = warp < nw && wa < we;
        const uint32_t len = plen[p];
        const unsigned char* src_lane = a.skew_codes + pso[p] * (32ull * M) + lane * 16;
        uint4 A[M / 16], B[M / 16];
        if (active) {
            load_tile<M>(A, src_lane, wa);
            load_tile<M>(B, src_lane, wa + 1);  // tile we (>= wa + 1) holds the range's tails
        }
        mbar_wait(bars + b, phase[b]);
        phase[b] ^= 1u;
        if (active) {
            const uint32_t lbase = plo[p];
            float cur = 0.0f, prev = 0.0f;
            for (uint32_t j = wa;; j += 2) {
                if (b == 0)
                    skew_round<M, 0>(A, bt, cur, prev, mk, nk, std::make_integer_sequence<int, M>{});
                else
                    skew_round<M, int(L::kImgStride)>(A, bt, cur, prev, mk, nk, std::make_integer_sequence<int, M>{});
                if (j + 2 <= we) load_tile<M>(A, src_lane, j + 2);
                {
                    const uint32_t e = (j - 1) * kTileEntries + lane;
                    const uint32_t key = __float_as_uint(prev);
                    topk_insert(t, key, j > wa && e < len && key <= t.thr, lbase + e, lane, k, a.ids);
                }
                prev = cur;
                cur = 0.0f;
                if (j + 1 > we) break;
                if (b == 0)
                    skew_round<M, 0>(B, bt, cur, prev, mk, nk, std::make_integer_sequence<int, M>{});
                else
                    skew_round<M, int(L::kImgStride)>(B, bt, cur, prev, mk, nk, std::make_integer_sequence<int, M>{});
                if (j + 3 <= we) load_tile<M>(B, src_lane, j + 3);
                {
                    const uint32_t e = j * kTileEntries + lane;
                    const uint32_t key = __float_as_uint(prev);
                    topk_insert(t, key, e < len && key <= t.thr, lbase + e, lane, k, a.ids);
                }
                prev = cur;
                cur = 0.0f;
                if (j + 2 > we) break;
            }
        }
        __syncthreads();  // every warp is done with buffer b
        uint32_t pn;
        if (next_segment(pn)) {
            seg_p[b] = pn;
            issue_image(b, pn);
            ++nseg;
        }
    }
    B1_MARK(6);
    // CTA top-k: k rounds of the smallest (key, id) among the warp list heads
    stash[warp * 64 + lane] = lane < k ? t.key : 0xffffffffu;
    stash[warp * 64 + 32 + lane] = t.pos;
    __syncthreads();
    if (warp == 0) {
        const uint32_t* ml = stash + lane * 64;
        const bool own = lane < uint32_t(kWarps);
        uint32_t hi = 0;
        uint32_t hk = own ? ml[0] : 0xffffffffu, hp = own ? ml[32] : 0u;
        uint32_t rk = 0xffffffffu, rp = 0u, cnt = 0;
        for (uint32_t r = 0; r < k; ++r) {
            const uint32_t kmin = __reduce_min_sync(0xffffffffu, hk);
            if (kmin == 0xffffffffu) break;
            const unsigned tie = __ballot_sync(0xffffffffu, hk == kmin);
            int win = __ffs(tie) - 1;
            if (tie & (tie - 1)) {  // exact distance tie between warps: lowest chunk id first
                uint64_t id = hk == kmin ? a.ids[hp] : ~0ull;
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const uint64_t oid = __shfl_xor_sync(0xffffffffu, id, o);
                    id = oid < id ? oid : id;
                }
                win = __ffs(__ballot_sync(0xffffffffu, hk == kmin && a.ids[hp] == id)) - 1;
            }
            const uint32_t wp = __shfl_sync(0xffffffffu, hp, win);
            if (lane == r) {
                rk = kmin;
                rp = wp;
            }
            ++cnt;
            if (int(lane) == win) {
                ++hi;
                hk = hi < k ? ml[hi] : 0xffffffffu;
                hp = hi < k ? ml[32 + hi] : 0u;
            }
        }
        a.cand_key[cta * 32 + lane] = lane < cnt ? rk : 0xffffffffu;
        a.cand_id[cta * 32 + lane] = lane < cnt ? a.ids[rp] : ~0ull;
    }

    // ----------------------------------------- 5. final merge (last CTA)
    __shared__ uint32_t s_last;
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        s_last = atomicAdd(a.sync + 2, 1u) == G - 1;
    }
    __syncthreads();
    B1_MARK(7);
    if (!s_last) return;
    __threadfence();
    if (tid == 0) {
        a.sync[2] = 0;  // ticket and barrier counter back to their start state
        a.sync[0] = 0;  // (every CTA has passed both barriers: it took a ticket)
        s_n = 0;
    }
    // one pass over the k meaningful slots of every CTA's list (sorted by
    // (distance, id)); U2 = the k-th smallest CTA head; keep what is <= U2
    __shared__ uint32_t s_uk;
    __shared__ uint64_t s_uid;
    if (tid == 0) {
        s_uk = 0xffffffffu;
        s_uid = ~0ull;
    }
    constexpr uint32_t kCpt = (kMaxGrid * 32 + kThreads - 1) / kThreads;
    const uint32_t ncand = G * k;
    uint32_t ckr[kCpt];
    uint64_t cir[kCpt];
#pragma unroll
    for (uint32_t u = 0; u < kCpt; ++u) {
        const uint32_t i = tid + u * kThreads;
        const uint32_t b = i / k, j = i - b * k;
        ckr[u] = i < ncand ? __ldcg(a.cand_key + b * 32 + j) : 0xffffffffu;
        cir[u] = i < ncand ? __ldcg(a.cand_id + b * 32 + j) : ~0ull;
    }
    uint32_t* hkey = probe;  // probe info is no longer needed: [G] head keys, ids in `heads`
#pragma unroll
    for (uint32_t u = 0; u < kCpt; ++u) {
        const uint32_t i = tid + u * kThreads;
        if (i < ncand && i % k == 0) {
            hkey[i / k] = ckr[u];
            heads[i / k] = cir[u];
        }
    }
    __syncthreads();
    for (uint32_t b = tid; b < G; b += kThreads) {
        const uint32_t hk = hkey[b];
        const uint64_t hi = heads[b];
        uint32_t r = 0;
        for (uint32_t i = 0; i < G; ++i) {
            const uint32_t ok = hkey[i];
            const uint64_t oi = heads[i];
            r += ok < hk || (ok == hk && oi < hi);
        }
        if (r == k - 1) {
            s_uk = hk;
            s_uid = hi;
        }
    }
    __syncthreads();
    const uint32_t uk = s_uk;
    const uint64_t uid = s_uid;
#pragma unroll
    for (uint32_t u = 0; u < kCpt; ++u) {
        const uint32_t x = ckr[u];
        const uint64_t xi = cir[u];
        if (x != 0xffffffffu && (x < uk || (x == uk && xi <= uid))) {
            const uint32_t pos = atomicAdd(&s_n, 1u);
            if (pos < kFinalCap) {
                skey32[pos] = x;
                sid[pos] = xi;
            }
        }
    }
    __syncthreads();
    const uint32_t nf = min(s_n, kFinalCap), nfp = pow2_ceil(nf);
    for (uint32_t i = nf + tid; i < nfp; i += kThreads) {
        skey32[i] = 0xffffffffu;
        sid[i] = ~0ull;
    }
    __syncthreads();
    bitonic_pairs(skey32, sid, nfp);
    const unsigned long long scanned = (unsigned long long)scal[0] | ((unsigned long long)scal[1] << 32);
    const uint32_t count = scanned < k ? uint32_t(scanned) : k;
    if (tid < count) {
        a.o_ids[tid] = sid[tid];
        a.o_dist[tid] = __uint_as_float(skey32[tid]);
    }
    if (tid == 0) {
        *a.o_count = count;
        if (a.o_scanned) *a.o_scanned = scanned;
    }
    B1_MARK(8);
}

}  // namespace

// Opt-in (PRAG_GPU_BATCH1=1): measured on B200 (tools/b1_time.py, config B,
// k = 2, back-to-back searches) the single launch takes 28.7 / 39.0 / 57.4 us
// at nprobe 1 / 16 / 64 against 27.9 / 33.8 / 46.5 us for the PDL-chained
// five kernels: the grid barriers and the per-phase memory round trips cost
// more than the launch boundaries they remove, so the chain stays the default.
static bool batch1_enabled() {
    const char* e = getenv("PRAG_GPU_BATCH1");
    return e != nullptr && e[0] == '1';
}

#ifdef PRAG_B1_TRACE
extern "C" int prag_gpu_debug_b1_trace(unsigned long long* out, size_t n) {
    return cudaMemcpyFromSymbol(out, g_b1_trace, (n < 256 * 16 ? n : 256 * 16) * 8) == cudaSuccess ? 0 : 3;
}
#endif

bool search1_eligible(const DeviceIndex& d, uint32_t nq, uint32_t nprobe, uint32_t k, int sms) {
    return nq == 1 && d.code_layout == 1 && (d.nsq == 32 || d.nsq == 64) && d.centroids4 && d.codewords &&
           d.d % 4 == 0 && k >= 1 && k <= 32 && nprobe >= 1 &&
           nprobe <= kMaxProbe && d.d <= kMaxD && d.sub_dim <= 16 && sms <= int(kMaxGrid) &&
           d.nlist <= uint64_t(sms) * kThreads && batch1_enabled();
}

size_t search1_scratch_bytes(const DeviceIndex& d, uint32_t nprobe, int grid) {
    const size_t stride = d.nsq == 64 ? B1Smem<64>::kImgStride : B1Smem<32>::kImgStride;
    Carver c{nullptr};
    c.take<uint64_t>(size_t(grid) * nprobe);
    c.take<unsigned char>(size_t(nprobe) * stride);
    c.take<uint4>(size_t(grid) * nprobe);
    c.take<uint32_t>(size_t(grid) * 32);
    c.take<uint64_t>(size_t(grid) * 32);
    return c.off + 256;
}

int launch_search1(const DeviceIndex& d, const float* dq, uint32_t nprobe, uint32_t k, uint64_t* o_ids,
                   float* o_dist, uint32_t* o_count, uint64_t* o_scanned, void* scratch, unsigned* sync, int grid,
                   cudaStream_t s) {
    const size_t stride = d.nsq == 64 ? B1Smem<64>::kImgStride : B1Smem<32>::kImgStride;
    Carver c{static_cast<char*>(scratch)};
    B1Args a{};
    a.centroids = d.centroids;
    a.centroids4 = reinterpret_cast<const float4*>(d.centroids4);
    a.codewords = d.codewords;
    a.list_len = d.list_len;
    a.list_off = d.list_off;
    a.skew_off = d.skew_off;
    a.skew_codes = d.skew_codes;
    a.ids = d.ids;
    a.nlist = d.nlist;
    a.d = d.d;
    a.sub = d.sub_dim;
    a.query = dq;
    a.nprobe = nprobe;
    a.k = k;
    a.o_ids = o_ids;
    a.o_dist = o_dist;
    a.o_count = o_count;
    a.o_scanned = o_scanned;
    a.coarse = c.take<uint64_t>(size_t(grid) * nprobe);
    a.images = c.take<unsigned char>(size_t(nprobe) * stride);
    a.caux = c.take<uint4>(size_t(grid) * nprobe);
    a.cand_key = c.take<uint32_t>(size_t(grid) * 32);
    a.cand_id = c.take<uint64_t>(size_t(grid) * 32);
    a.sync = sync;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // the grid barriers need every CTA resident
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (d.nsq == 32) {
        cfg.dynamicSmemBytes = B1Smem<32>::bytes;
        PG_CUDA(ensure_smem(reinterpret_cast<const void*>(search1_kernel<32>), B1Smem<32>::bytes));
        PG_CUDA(cudaLaunchKernelEx(&cfg, search1_kernel<32>, a));
    } else {
        cfg.dynamicSmemBytes = B1Smem<64>::bytes;
        PG_CUDA(ensure_smem(reinterpret_cast<const void*>(search1_kernel<64>), B1Smem<64>::bytes));
        PG_CUDA(cudaLaunchKernelEx(&cfg, search1_kernel<64>, a));
    }
    return PRAG_GPU_OK;
}

}  // namespace pg
