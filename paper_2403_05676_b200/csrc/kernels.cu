// kernels.cu -- sm_100a kernels of the IVF-PQ search path.
//
// Arithmetic contract: every distance is the
// reference's strictly sequential IEEE fp32 fold (common.hpp:73-80,
// annindex.hpp:279, :292-302) built from __fsub_rn/__fmul_rn/__fadd_rn so
// nvcc can never contract to FFMA or reassociate; results are bit-identical to
// the x86-64 SSE reference. Selection is exact on the (distance, id) total
// order of annindex.hpp:55-58 / :281.
//
// Kernels (one batch of nq queries):
//   K1  coarse_exact_kernel     q x centroid distances          annindex.hpp:277-280
//   K1b select_kernel<Probe>    per-query top-nprobe            annindex.hpp:281
//   P   plan_kernel             (q, list, tile) work items + scanned_vectors :284-305
//   K2+K3 scan_kernel           LUT in SMEM + list scan         :285-305
//   K4  select_kernel<Final>    per-query top-k                 :313, :54-60
//   K5  merge_kernel            shard merge (multi-GPU)
#include <cstdint>

#include "internal.h"

namespace pg {

namespace {

constexpr int kSelThreads = 1024;
constexpr uint32_t kSortCap = 2048;   // elements sorted in SMEM; larger k sorts in global scratch
constexpr int kPoolThreads = 256;     // select_pool CTA
constexpr uint32_t kPoolCap = 2048;   // select_pool: survivors kept in SMEM
constexpr uint32_t kChunk = 4096;     // entries per scan work item

// Monotone float -> uint32 map (total order == float order for non-NaN).
__device__ __forceinline__ uint32_t ord_key(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_float(uint32_t k) {
    uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(u);
}

// ------------------------------------------------------------------ K1
// One thread = one centroid x QB queries. Centroids are read transposed
// ([d][nlist], coalesced across the warp); query rows sit in SMEM and are
// warp-broadcast. Each (q, c) accumulator is the sequential fold of
// squared_l2(query, centroid, d) (common.hpp:73-80): diff = q - c.
template <int QB>
__global__ void __launch_bounds__(128) coarse_exact_kernel(const float* __restrict__ centT,
                                                           const float* __restrict__ queries,
                                                           uint32_t nq, uint32_t nlist, uint32_t d,
                                                           float* __restrict__ out) {
    extern __shared__ float sq[];  // [QB][d]
    const uint32_t q0 = blockIdx.y * QB;
    for (uint32_t i = threadIdx.x; i < QB * d; i += blockDim.x) {
        uint32_t qi = i / d, j = i - qi * d;
        sq[i] = (q0 + qi < nq) ? queries[size_t(q0 + qi) * d + j] : 0.0f;
    }
    __syncthreads();
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nlist) return;
    float acc[QB];
#pragma unroll
    for (int qi = 0; qi < QB; ++qi) acc[qi] = 0.0f;
    const float* col = centT + c;
#pragma unroll 4
    for (uint32_t j = 0; j < d; ++j) {
        const float cv = __ldg(col + size_t(j) * nlist);
#pragma unroll
        for (int qi = 0; qi < QB; ++qi) {
            const float diff = __fsub_rn(sq[qi * d + j], cv);
            acc[qi] = __fadd_rn(acc[qi], __fmul_rn(diff, diff));
        }
    }
#pragma unroll
    for (int qi = 0; qi < QB; ++qi)
        if (q0 + qi < nq) out[size_t(q0 + qi) * nlist + c] = acc[qi];
}

// Same fold, vectorised for d % 4 == 0: centroids as float4 per thread from
// [d/4][nlist] (one LDG.128 per 4 dims), queries as [d][4] in SMEM (one
// LDS.128 broadcast per dim), q - c for two queries per FADD2 (exact: one
// rounding per difference); squares and the fold stay scalar FMUL/FADD.
__device__ __forceinline__ void sub2_bc(float a0, float a1, float b, float& d0, float& d1) {
    unsigned long long out;
    asm("{.reg .b64 A, B;\n"
        " mov.b64 A, {%1, %2};\n"
        " mov.b64 B, {%3, %3};\n"
        " sub.rn.f32x2 %0, A, B;}"
        : "=l"(out)
        : "f"(a0), "f"(a1), "f"(b));
    d0 = __uint_as_float(uint32_t(out));
    d1 = __uint_as_float(uint32_t(out >> 32));
}

// Thread = one centroid x 2 queries (more warps than a wider query block:
// the kernel is latency-bound on the centroid stream from L2).
__global__ void __launch_bounds__(128) coarse_exact4_kernel(const float4* __restrict__ cent4,
                                                            const float* __restrict__ queries, uint32_t nq,
                                                            uint32_t nlist, uint32_t d, float* __restrict__ out) {
    extern __shared__ __align__(16) float sq2[];  // [d][2]
    const uint32_t q0 = blockIdx.y * 2;
    for (uint32_t i = threadIdx.x; i < 2 * d; i += blockDim.x) {
        const uint32_t qi = i & 1u, j = i >> 1;
        sq2[i] = (q0 + qi < nq) ? queries[size_t(q0 + qi) * d + j] : 0.0f;
    }
    __syncthreads();
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nlist) return;
    float a0 = 0.0f, a1 = 0.0f;
    const float4* colp = cent4 + c;
    const uint32_t d4 = d >> 2;
#pragma unroll 8
    for (uint32_t jj = 0; jj < d4; ++jj) {
        const float4 cv = __ldg(colp + size_t(jj) * nlist);
        const float4 qa = *reinterpret_cast<const float4*>(sq2 + jj * 8);      // dims 4jj, 4jj+1
        const float4 qb = *reinterpret_cast<const float4*>(sq2 + jj * 8 + 4);  // dims 4jj+2, 4jj+3
        float d0, d1;
        sub2_bc(qa.x, qa.y, cv.x, d0, d1);
        a0 = __fadd_rn(a0, __fmul_rn(d0, d0));
        a1 = __fadd_rn(a1, __fmul_rn(d1, d1));
        sub2_bc(qa.z, qa.w, cv.y, d0, d1);
        a0 = __fadd_rn(a0, __fmul_rn(d0, d0));
        a1 = __fadd_rn(a1, __fmul_rn(d1, d1));
        sub2_bc(qb.x, qb.y, cv.z, d0, d1);
        a0 = __fadd_rn(a0, __fmul_rn(d0, d0));
        a1 = __fadd_rn(a1, __fmul_rn(d1, d1));
        sub2_bc(qb.z, qb.w, cv.w, d0, d1);
        a0 = __fadd_rn(a0, __fmul_rn(d0, d0));
        a1 = __fadd_rn(a1, __fmul_rn(d1, d1));
    }
    out[size_t(q0) * nlist + c] = a0;
    if (q0 + 1 < nq) out[size_t(q0 + 1) * nlist + c] = a1;
}

// ------------------------------------------------- block-wide exact top-k
// Selects the kk = min(k, n) smallest (key, tie) pairs of a candidate set
// (keys from ord_key(distance), tie = list id or chunk_id) and writes them
// sorted ascending. Radix select on the 32-bit key (4 x 8-bit digits), then
// if the k-th key is shared, radix select on the 64-bit tie among the equal
// keys; the selected set is then bitonic-sorted on (key, tie).
struct SelShared {
    uint32_t hist[256];
    uint32_t prefix, rank, eq_count, nsel;
    uint64_t tie_prefix;
    uint32_t skey[kSortCap];
    uint64_t stie[kSortCap];
};


__device__ __forceinline__ void warp_hist_add(uint32_t* hist, uint32_t bucket, bool active) {
    // Warp-aggregated shared-memory histogram increment (distances share
    // their top digits, so plain atomics would serialise on one bin).
    const unsigned amask = __ballot_sync(0xffffffffu, active);
    if (!active) return;
    const unsigned peers = __match_any_sync(amask, bucket);
    const int leader = __ffs(peers) - 1;
    if ((threadIdx.x & 31) == leader) atomicAdd(&hist[bucket], __popc(peers));
}

// After a histogram pass: find the bucket holding the rank-th element
// (1-based) and update prefix/rank. Executed by warp 0.
__device__ __forceinline__ void hist_pick(SelShared& sm, int shift, bool tie_pass) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    uint32_t v[8];
    uint32_t local = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        v[i] = sm.hist[lane * 8 + i];
        local += v[i];
    }
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    const uint32_t excl = incl - local;
    const uint32_t rank = sm.rank;
    const bool mine = excl < rank && rank <= incl;
    if (mine) {
        uint32_t c = excl;
        int b = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (c + v[i] >= rank) {
                b = i;
                break;
            }
            c += v[i];
        }
        const uint32_t bucket = lane * 8 + b;
        sm.rank = rank - c;
        sm.eq_count = v[b];
        if (tie_pass)
            sm.tie_prefix |= uint64_t(bucket) << shift;
        else
            sm.prefix |= bucket << shift;
    }
}

template <class Src>
__device__ void block_topk(const Src& src, uint32_t n, uint32_t k, SelShared& sm, uint32_t* gkey,
                           uint64_t* gtie, float* out_dist, uint64_t* out_tie, uint32_t* out_count) {
    const uint32_t kk = n < k ? n : k;
    const uint32_t tid = threadIdx.x, nth = blockDim.x;
    bool use_tie = false;
    uint32_t T = 0xffffffffu;
    uint64_t TI = ~0ull;
    if (n > k) {
        if (tid == 0) {
            sm.prefix = 0;
            sm.rank = k;
            sm.tie_prefix = 0;
        }
        uint32_t mask = 0;
        for (int shift = 24; shift >= 0; shift -= 8) {
            for (uint32_t i = tid; i < 256; i += nth) sm.hist[i] = 0;
            __syncthreads();
            const uint32_t prefix = sm.prefix;
            for (uint32_t base = 0; base < n; base += nth) {
                const uint32_t i = base + tid;
                uint32_t key = 0;
                bool act = false;
                if (i < n) {
                    key = src.key(i);
                    act = (key & mask) == prefix;
                }
                warp_hist_add(sm.hist, (key >> shift) & 255u, act);
            }
            __syncthreads();
            hist_pick(sm, shift, false);
            __syncthreads();
            mask |= 0xffu << shift;
        }
        T = sm.prefix;
        // sm.rank = how many of the key==T elements are needed; eq_count = how many exist
        if (sm.eq_count > sm.rank) {
            use_tie = true;
            uint64_t tmask = 0;
            for (int shift = 56; shift >= 0; shift -= 8) {
                for (uint32_t i = tid; i < 256; i += nth) sm.hist[i] = 0;
                __syncthreads();
                const uint64_t tp = sm.tie_prefix;
                for (uint32_t base = 0; base < n; base += nth) {
                    const uint32_t i = base + tid;
                    uint64_t tie = 0;
                    bool act = false;
                    if (i < n && src.key(i) == T) {
                        tie = src.tie(i);
                        act = (tie & tmask) == tp;
                    }
                    warp_hist_add(sm.hist, uint32_t(tie >> shift) & 255u, act);
                }
                __syncthreads();
                hist_pick(sm, shift, true);
                __syncthreads();
                tmask |= uint64_t(0xff) << shift;
            }
            TI = sm.tie_prefix;
        }
    }
    // gather the selected set
    uint32_t pw = 1;
    while (pw < kk) pw <<= 1;
    const bool in_smem = pw <= kSortCap;
    uint32_t* keys = in_smem ? sm.skey : gkey;
    uint64_t* ties = in_smem ? sm.stie : gtie;
    if (tid == 0) sm.nsel = 0;
    __syncthreads();
    for (uint32_t base = 0; base < n; base += nth) {
        const uint32_t i = base + tid;
        bool take = false;
        uint32_t key = 0;
        uint64_t tie = 0;
        if (i < n) {
            key = src.key(i);
            if (key < T || (n <= k)) {
                take = true;
            } else if (key == T) {
                tie = src.tie(i);
                take = !use_tie || tie <= TI;
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        uint32_t wbase = 0;
        if ((tid & 31) == 0 && bal) wbase = atomicAdd(&sm.nsel, __popc(bal));
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
        if (take) {
            const uint32_t pos = wbase + __popc(bal & ((1u << (tid & 31)) - 1));
            if (pos < kk) {  // duplicate (key, tie) pairs can exceed kk; they are interchangeable
                if (key != T || n <= k) tie = src.tie(i);
                keys[pos] = key;
                ties[pos] = tie;
            }
        }
    }
    __syncthreads();
    for (uint32_t i = kk + tid; i < pw; i += nth) {
        keys[i] = 0xffffffffu;
        ties[i] = ~0ull;
    }
    __syncthreads();
    // bitonic sort on (key, tie), ascending
    for (uint32_t size = 2; size <= pw; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = tid; t < pw / 2; t += nth) {
                const uint32_t lo = 2 * t - (t & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint32_t ka = keys[lo], kb = keys[hi];
                const uint64_t ta = ties[lo], tb = ties[hi];
                const bool gt = ka > kb || (ka == kb && ta > tb);
                if (gt == up) {
                    keys[lo] = kb;
                    keys[hi] = ka;
                    ties[lo] = tb;
                    ties[hi] = ta;
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = tid; i < kk; i += nth) {
        if (out_dist) out_dist[i] = key_float(keys[i]);
        out_tie[i] = ties[i];
    }
    if (tid == 0 && out_count) *out_count = kk;
    __syncthreads();
}

struct ProbeSrc {
    const float* d;
    __device__ uint32_t key(uint32_t i) const { return ord_key(d[i]); }
    __device__ uint64_t tie(uint32_t i) const { return i; }
};

struct FinalSrc {
    const float* d;
    const uint32_t* entry;
    const uint64_t* ids;
    __device__ uint32_t key(uint32_t i) const { return ord_key(d[i]); }
    __device__ uint64_t tie(uint32_t i) const { return ids[entry[i]]; }
};

struct MergeSrc {
    const uint32_t* k;
    const uint64_t* t;
    __device__ uint32_t key(uint32_t i) const { return k[i]; }
    __device__ uint64_t tie(uint32_t i) const { return t[i]; }
};

// K1b: per-query top-nprobe lists, (distance, list id) order (annindex.hpp:281).
__global__ void __launch_bounds__(kSelThreads) select_probe_kernel(const float* __restrict__ coarse,
                                                                   uint32_t nlist, uint32_t nprobe,
                                                                   uint32_t* __restrict__ probe,
                                                                   float* __restrict__ probe_dist,
                                                                   uint32_t* gkey, uint64_t* gtie) {
    extern __shared__ __align__(16) unsigned char smraw[];
    SelShared& sm = *reinterpret_cast<SelShared*>(smraw);
    const uint32_t q = blockIdx.x;
    ProbeSrc src{coarse + size_t(q) * nlist};
    uint32_t pw = 1;
    while (pw < nprobe) pw <<= 1;
    uint64_t* ties = gtie + size_t(q) * pw;
    block_topk(src, nlist, nprobe, sm, gkey + size_t(q) * pw, ties, probe_dist + size_t(q) * nprobe,
               ties, nullptr);
    // ties[] now holds the sorted list ids; narrow to u32
    for (uint32_t i = threadIdx.x; i < nprobe; i += blockDim.x) probe[size_t(q) * nprobe + i] = uint32_t(ties[i]);
}

// ------------------------------------------------------------------- plan
// One CTA. For each (q, p) pair: len = |list|, its candidate slot offset and
// ceil(len / kChunk) work items {q, list, begin, out_off}. Per-query
// scanned_vectors is the sum of probed list lengths (annindex.hpp:305);
// empty lists contribute nothing (:290).
template <typename T>
__device__ T block_excl_scan(T v, T* warp_tmp, T& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tmp[w] = incl;
    __syncthreads();
    if (w == 0) {
        T x = lane < nw ? warp_tmp[lane] : T(0);
        T xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += t;
        }
        if (lane < nw) warp_tmp[lane] = xi - x;
        if (lane == nw - 1) warp_tmp[32] = xi;
    }
    __syncthreads();
    T res = warp_tmp[w] + incl - v;
    total = warp_tmp[32];
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(1024) plan_kernel(const uint32_t* __restrict__ probe,
                                                    const uint32_t* __restrict__ list_len, uint32_t nq,
                                                    uint32_t nprobe, uint64_t* __restrict__ q_cand_off,
                                                    uint64_t* __restrict__ scanned, uint4* __restrict__ items,
                                                    uint32_t* __restrict__ num_items,
                                                    uint32_t* __restrict__ cursor, uint64_t item_cap) {
    __shared__ uint64_t tmp64[33];
    __shared__ uint32_t tmp32[33];
    const uint32_t P = nq * nprobe;
    uint64_t carry_c = 0;
    uint32_t carry_i = 0;
    for (uint32_t base = 0; base < P; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const bool valid = i < P;
        const uint32_t list = valid ? probe[i] : 0;
        const uint32_t len = valid ? list_len[list] : 0;
        const uint32_t nit = (len + kChunk - 1) / kChunk;
        uint64_t tot_c;
        uint32_t tot_i;
        const uint64_t ec = block_excl_scan<uint64_t>(len, tmp64, tot_c);
        const uint32_t ei = block_excl_scan<uint32_t>(nit, tmp32, tot_i);
        if (valid) {
            const uint32_t q = i / nprobe, p = i - q * nprobe;
            if (p == 0) q_cand_off[q] = carry_c + ec;
            for (uint32_t j = 0; j < nit; ++j) {
                const uint64_t slot = carry_i + ei + j;
                if (slot < item_cap)
                    items[slot] = make_uint4(q, list, j * kChunk, uint32_t(carry_c + ec + uint64_t(j) * kChunk));
            }
        }
        carry_c += tot_c;
        carry_i += tot_i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        q_cand_off[nq] = carry_c;
        *num_items = carry_i;
        *cursor = 0;
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) scanned[q] = q_cand_off[q + 1] - q_cand_off[q];
}

// ---------------------------------------------------------------- K2 + K3
// Persistent CTAs pull (q, list, begin) work items. On a new (q, list):
// residual r = q - c_list (annindex.hpp:292) and the ADC table
// T[sq][code] = squared_l2(r_sq, w[sq][code], sub_dim) (:293-299) are built
// in SMEM; then each thread folds one entry at a time:
// dist = ((0 + T[0][c0]) + T[1][c1]) + ... (:300-302).
// Code byte b of entry e of a list in the lane-skewed tile layout K3 reads
// (scan_skew.cu): lane t = e mod 32 of tile e / 32 folds it at step b + t;
// steps past m continue in the next tile, whose tail bytes m = 64 stores as
// code + 1 (scan_skew.cu SkewSmem).
__device__ __forceinline__ uint32_t skew_code(const uint8_t* __restrict__ tiles, uint32_t nsq, uint32_t e,
                                              uint32_t b) {
    const uint32_t t = e & 31u;
    uint32_t tile = e >> 5, s = b + t;
    bool tail = false;
    if (s >= nsq) {
        s -= nsq;
        ++tile;
        tail = true;
    }
    const uint32_t v = tiles[size_t(tile) * 32 * nsq + (s >> 4) * 512 + t * 16 + (s & 15u)];
    return (tail && nsq == 64) ? ((v - 1) & 255u) : v;
}

// kSkew: the index keeps only the lane-skewed code tiles (m = 32 / 64); the
// entry's code bytes are gathered from them instead of the plain array.
template <bool kSmemLut, bool kSkew>
__global__ void __launch_bounds__(256) scan_kernel(
    const float* __restrict__ queries, const float* __restrict__ centroids,
    const float* __restrict__ codewordsT, const uint64_t* __restrict__ list_off,
    const uint32_t* __restrict__ list_len, const uint8_t* __restrict__ codes, const uint64_t* __restrict__ skew_off,
    uint32_t d, uint32_t nsq, uint32_t sub_dim, const uint4* __restrict__ items,
    const uint32_t* __restrict__ num_items, uint32_t* __restrict__ cursor, float* __restrict__ cand_dist,
    uint32_t* __restrict__ cand_entry, float* __restrict__ glut) {
    extern __shared__ __align__(16) float smf[];
    float* resid = smf;                                   // [d]
    float* lut = kSmemLut ? smf + ((d + 3) & ~3u) : glut + size_t(blockIdx.x) * nsq * 256;
    __shared__ uint32_t s_item;
    const uint32_t total = *num_items;
    uint32_t cur_q = 0xffffffffu, cur_list = 0xffffffffu;
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(cursor, 1u);
        __syncthreads();
        const uint32_t it = s_item;
        if (it >= total) break;
        const uint4 w = items[it];
        const uint32_t q = w.x, list = w.y, begin = w.z, out_off = w.w;
        if (q != cur_q || list != cur_list) {
            const float* qv = queries + size_t(q) * d;
            const float* cv = centroids + size_t(list) * d;
            for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) resid[j] = __fsub_rn(qv[j], cv[j]);
            __syncthreads();
            for (uint32_t t = threadIdx.x; t < nsq * 256; t += blockDim.x) {
                const uint32_t s = t >> 8, code = t & 255u;
                const float* r = resid + s * sub_dim;
                const float* wv = codewordsT + size_t(s) * sub_dim * 256 + code;
                float acc = 0.0f;
                for (uint32_t j = 0; j < sub_dim; ++j) {
                    const float diff = __fsub_rn(r[j], __ldg(wv + j * 256));
                    acc = __fadd_rn(acc, __fmul_rn(diff, diff));
                }
                lut[t] = acc;
            }
            cur_q = q;
            cur_list = list;
            __syncthreads();
        }
        const uint32_t len = list_len[list];
        const uint32_t end = min(len, begin + kChunk);
        const uint64_t lbase = list_off[list];
        for (uint32_t e = begin + threadIdx.x; e < end; e += blockDim.x) {
            const uint64_t slot = lbase + e;
            const uint8_t* c = codes + slot * nsq;
            float dist = 0.0f;
            if (kSkew) {
                const uint8_t* tiles = codes + skew_off[list] * 32 * nsq;
                for (uint32_t s = 0; s < nsq; ++s) dist = __fadd_rn(dist, lut[s * 256 + skew_code(tiles, nsq, e, s)]);
            } else if ((nsq & 3u) == 0) {
                for (uint32_t s4 = 0; s4 < nsq; s4 += 4) {
                    const uint32_t wd = *reinterpret_cast<const uint32_t*>(c + s4);
                    dist = __fadd_rn(dist, lut[(s4 + 0) * 256 + (wd & 255u)]);
                    dist = __fadd_rn(dist, lut[(s4 + 1) * 256 + ((wd >> 8) & 255u)]);
                    dist = __fadd_rn(dist, lut[(s4 + 2) * 256 + ((wd >> 16) & 255u)]);
                    dist = __fadd_rn(dist, lut[(s4 + 3) * 256 + (wd >> 24)]);
                }
            } else {
                for (uint32_t s = 0; s < nsq; ++s) dist = __fadd_rn(dist, lut[s * 256 + c[s]]);
            }
            const uint32_t o = out_off + (e - begin);
            cand_dist[o] = dist;
            cand_entry[o] = uint32_t(slot);
        }
        __syncthreads();
    }
}

// K4: per-query exact top-k over all candidates of the query.
__global__ void __launch_bounds__(kSelThreads) select_final_kernel(
    const float* __restrict__ cand_dist, const uint32_t* __restrict__ cand_entry,
    const uint64_t* __restrict__ ids, const uint64_t* __restrict__ q_cand_off, uint32_t k,
    uint64_t* __restrict__ out_ids, float* __restrict__ out_dist, uint32_t* __restrict__ out_count,
    uint32_t* gkey, uint64_t* gtie, uint32_t pw) {
    extern __shared__ __align__(16) unsigned char smraw[];
    SelShared& sm = *reinterpret_cast<SelShared*>(smraw);
    const uint32_t q = blockIdx.x;
    const uint64_t b = q_cand_off[q], e = q_cand_off[q + 1];
    FinalSrc src{cand_dist + b, cand_entry + b, ids};
    block_topk(src, uint32_t(e - b), k, sm, gkey + size_t(q) * pw, gtie + size_t(q) * pw,
               out_dist + size_t(q) * k, out_ids + size_t(q) * k, out_count + q);
}

// K5: exact top-k of the union of per-shard top-k lists.
__global__ void __launch_bounds__(kSelThreads) merge_kernel(
    const uint64_t* __restrict__ ids, const float* __restrict__ dist, const uint32_t* __restrict__ count,
    const uint64_t* __restrict__ scanned, uint32_t nparts, uint32_t nq, uint32_t kin, uint32_t k,
    uint64_t* __restrict__ out_ids, float* __restrict__ out_dist, uint32_t* __restrict__ out_count,
    uint64_t* __restrict__ out_scanned, uint32_t* ckey, uint64_t* ctie, uint32_t* gkey, uint64_t* gtie,
    uint32_t pw) {
    extern __shared__ __align__(16) unsigned char smraw[];
    SelShared& sm = *reinterpret_cast<SelShared*>(smraw);
    __shared__ uint32_t s_n;
    const uint32_t q = blockIdx.x;
    const size_t cap = size_t(nparts) * kin;
    uint32_t* ck = ckey + q * cap;
    uint64_t* ct = ctie + q * cap;
    if (threadIdx.x == 0) {
        uint32_t n = 0;
        uint64_t sc = 0;
        for (uint32_t p = 0; p < nparts; ++p) {
            const uint32_t c = min(count[size_t(p) * nq + q], kin);
            n += c;
            if (scanned) sc += scanned[size_t(p) * nq + q];
        }
        s_n = n;
        if (out_scanned) out_scanned[q] = sc;
    }
    __syncthreads();
    // compact valid entries (per part, the first count[p][q] of kin slots)
    for (uint32_t p = 0; p < nparts; ++p) {
        uint32_t before = 0;
        for (uint32_t pp = 0; pp < p; ++pp) before += min(count[size_t(pp) * nq + q], kin);
        const uint32_t c = min(count[size_t(p) * nq + q], kin);
        const size_t src = (size_t(p) * nq + q) * kin;
        for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
            ck[before + i] = ord_key(dist[src + i]);
            ct[before + i] = ids[src + i];
        }
    }
    __syncthreads();
    MergeSrc s{ck, ct};
    block_topk(s, s_n, k, sm, gkey + size_t(q) * pw, gtie + size_t(q) * pw, out_dist + size_t(q) * k,
               out_ids + size_t(q) * k, out_count + q);
}

// K4 helper: more survivors than threads. The min(k, c)-th smallest key K of
// vkey[0, c) by a 4-pass radix select (8 bits per pass, SMEM histogram), then
// the survivors with key <= K (k of them plus any distance ties at K) are
// compacted to the front of vkey / vid; returns their count. Whole block.
__device__ __noinline__ uint32_t narrow_survivors(uint32_t* vkey, uint64_t* vid, uint32_t c, uint32_t k,
                                                  uint32_t* nsurv) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t sel[2];  // selected key prefix, rank still to find within it
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    if (tid == 0) {
        sel[0] = 0;
        sel[1] = min(k, c);
    }
    uint32_t mask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t b = tid; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const uint32_t prefix = sel[0];
        for (uint32_t i = tid; i < c; i += blockDim.x) {
            const uint32_t key = vkey[i];
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            uint32_t v[8], local = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                v[i] = hist[lane * 8 + i];
                local += v[i];
            }
            uint32_t incl = local;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= uint32_t(o)) incl += t;
            }
            const uint32_t r = sel[1];
            __syncwarp();
            uint32_t acc = incl - local;
            if (acc < r && r <= incl) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (acc + v[i] >= r) {
                        sel[0] = prefix | ((lane * 8u + uint32_t(i)) << shift);
                        sel[1] = r - acc;
                        break;
                    }
                    acc += v[i];
                }
            }
        }
        __syncthreads();
        mask |= 255u << shift;
    }
    const uint32_t K = sel[0];
    constexpr int kPer = int(kPoolCap / kPoolThreads);
    uint32_t kk[kPer];
    uint64_t ii[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const uint32_t i = uint32_t(u) * blockDim.x + tid;
        kk[u] = i < c ? vkey[i] : 0xffffffffu;
        ii[u] = i < c ? vid[i] : ~0ull;
    }
    if (tid == 0) *nsurv = 0;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const bool take = kk[u] <= K;
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        uint32_t base = 0;
        if (lane == 0 && bal) base = atomicAdd(nsurv, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (take) {
            const uint32_t pos = base + __popc(bal & ((1u << lane) - 1));
            vkey[pos] = kk[u];
            vid[pos] = ii[u];
        }
    }
    __syncthreads();
    return *nsurv;
}

// K4 (fast path): exact top-k of a query's candidate pool. The fused scan
// leaves, per work item, the CTA's exact top-k of that item as (key, entry
// slot) pairs (k slots, +inf
// sentinels), so a query's pool is k x its item count, contiguous. The CTA
// keeps the keys <= the query's final shared threshold T0 (some item left k
// candidates <= T0, so every top-k member is <= T0) in SMEM; up to one per
// thread (about k in practice; more are first narrowed to the keys <= the
// k-th smallest by a radix select), each survivor's rank by (distance,
// chunk_id) (annindex.hpp:54-60) is counted against the others and it is
// written to that output slot; otherwise (ties beyond the block, or more than
// kPoolCap survivors) one warp runs an exact insertion top-k, streaming the
// whole pool past kPoolCap. count = min(scanned_vectors, k) (annindex.hpp:313).
__global__ void __launch_bounds__(kPoolThreads) select_pool_kernel(
    const uint32_t* __restrict__ pool_key, const uint64_t* __restrict__ pool_id, const uint64_t* __restrict__ ids,
    const uint64_t* __restrict__ scanned, const uint32_t* __restrict__ q_item_off, const uint32_t* __restrict__ gthr,
    uint32_t k, uint64_t* __restrict__ out_ids, float* __restrict__ out_dist, uint32_t* __restrict__ out_count) {
    __shared__ __align__(16) uint32_t vkey[kPoolCap + 4];  // + padding for the 4-wide rank loop
    __shared__ uint64_t vid[kPoolCap];
    __shared__ uint32_t nsurv;
    CT_BEGIN;
    const uint32_t q = blockIdx.x, tid = threadIdx.x, lane = tid & 31u;
    size_t off;
    uint32_t n, total, T0, c;
    // Pass 0 runs the same code on four dummy keys with no global reads or
    // writes before waiting on K3 (this grid launches when K3 runs out of
    // work items): it pulls the instruction lines in while K3 drains.
    for (int pass = 0; pass < 2; ++pass) {
        const bool dry = pass == 0;
        if (!dry) {
            pdl_wait();  // the pool (and its offsets, from the planner) come from earlier kernels
            CT_WAITED(5);
        }
        off = dry ? 0 : size_t(q_item_off[q]) * k;
        n = dry ? 4u : (q_item_off[q + 1] - q_item_off[q]) * k;
        total = dry ? 0u : uint32_t(min(scanned[q], uint64_t(k)));
        const uint32_t graw = dry ? 0xffffffffu : gthr[q];  // raw distance bits (distances are >= 0); the pool holds ord_key()s
        T0 = graw != 0xffffffffu ? ord_key(__uint_as_float(graw)) : 0xfffffffeu;
        if (tid == 0) nsurv = 0;
        __syncthreads();
        for (uint32_t b0 = 0; b0 < n; b0 += 4 * kPoolThreads) {
            uint32_t key[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t i = b0 + u * kPoolThreads + tid;
                key[u] = i < n ? (dry ? i : pool_key[off + i]) : 0xffffffffu;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t i = b0 + u * kPoolThreads + tid;
                const bool take = key[u] <= T0;  // also drops the +inf sentinels and the tail
                const unsigned bal = __ballot_sync(0xffffffffu, take);
                uint32_t base = 0;
                if (lane == 0 && bal) base = atomicAdd(&nsurv, __popc(bal));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (take) {
                    const uint32_t pos = base + __popc(bal & ((1u << lane) - 1));
                    if (pos < kPoolCap) {
                        vkey[pos] = key[u];
                        vid[pos] = dry ? 0ull : ids[pool_id[off + i]];  // the pool holds entry slots
                    }
                }
            }
        }
        __syncthreads();
        c = nsurv;
        if (c > uint32_t(kPoolThreads) && c <= kPoolCap) c = narrow_survivors(vkey, vid, c, k, &nsurv);
        if (c <= uint32_t(kPoolThreads)) {
            // few survivors (the usual case: about k): each one's rank by (distance,
            // chunk id) among them, counted by its own thread, four keys per LDS.128
            if (tid < 4) vkey[c + tid] = 0xffffffffu;  // above every survivor (all <= T0 < 0xffffffff)
            __syncthreads();
            if (tid < c) {
                const uint32_t mk = vkey[tid];
                const uint64_t mi = vid[tid];
                uint32_t r = 0;
                for (uint32_t j = 0; j < c; j += 4) {
                    const uint4 kj = *reinterpret_cast<const uint4*>(vkey + j);
                    r += uint32_t(kj.x < mk) + uint32_t(kj.y < mk) + uint32_t(kj.z < mk) + uint32_t(kj.w < mk);
                    if (kj.x == mk || kj.y == mk || kj.z == mk || kj.w == mk) {  // distance ties: by chunk id
                        r += uint32_t(kj.x == mk && vid[j] < mi) + uint32_t(kj.y == mk && vid[j + 1] < mi) +
                             uint32_t(kj.z == mk && vid[j + 2] < mi) + uint32_t(kj.w == mk && vid[j + 3] < mi);
                    }
                }
                if (r < total) {
                    out_dist[size_t(q) * k + r] = key_float(mk);
                    out_ids[size_t(q) * k + r] = mi;
                }
            } else if (tid < total) {  // fewer survivors than results: unfilled slots
                out_dist[size_t(q) * k + tid] = key_float(0xffffffffu);
                out_ids[size_t(q) * k + tid] = ~0ull;
            }
            if (dry) {
                __syncthreads();  // vkey / nsurv are reused by the real pass
                continue;
            }
            if (tid == 0) out_count[q] = total;
            CT_END(5);
            return;
        }
        break;
    }
    if (tid >= 32) {
        CT_END(5);
        return;
    }
    const bool from_smem = c <= kPoolCap;
    const uint32_t m = from_smem ? c : n;
    // lane r holds the r-th best (key, id); (thk, thid) is the k-th
    uint32_t lk = 0xffffffffu, thk = 0xffffffffu;
    uint64_t lid = ~0ull, thid = ~0ull;
    for (uint32_t i0 = 0; i0 < m; i0 += 32) {
        const uint32_t i = i0 + lane;
        uint32_t key = 0xffffffffu;
        if (i < m) key = from_smem ? vkey[i] : pool_key[off + i];
        const bool pre = key <= min(T0, thk);
        unsigned bal = __ballot_sync(0xffffffffu, pre);
        if (!bal) continue;
        const uint64_t id = pre ? (from_smem ? vid[i] : ids[pool_id[off + i]]) : ~0ull;
        while (bal) {
            const int src = __ffs(bal) - 1;
            bal &= bal - 1;
            const uint32_t ck = __shfl_sync(0xffffffffu, key, src);
            const uint64_t cid = __shfl_sync(0xffffffffu, id, src);
            if (ck > thk || (ck == thk && cid >= thid)) continue;
            const unsigned gm = __ballot_sync(0xffffffffu, lk > ck || (lk == ck && lid > cid));
            const int pos = gm ? __ffs(gm) - 1 : 32;
            const uint32_t uk = __shfl_up_sync(0xffffffffu, lk, 1);
            const uint64_t ui = __shfl_up_sync(0xffffffffu, lid, 1);
            if (int(lane) > pos) {
                lk = uk;
                lid = ui;
            } else if (int(lane) == pos) {
                lk = ck;
                lid = cid;
            }
            thk = __shfl_sync(0xffffffffu, lk, k - 1);
            thid = __shfl_sync(0xffffffffu, lid, k - 1);
        }
    }
    if (lane < total) {
        out_dist[size_t(q) * k + lane] = key_float(lk);
        out_ids[size_t(q) * k + lane] = lid;
    }
    if (lane == 0) out_count[q] = total;
    CT_END(5);
}

}  // namespace

#ifdef PRAG_CHAIN_TRACE
CT_BIND_FN(ct_bind_kernels)
#endif

int launch_select_pool(const uint32_t* pool_key, const uint64_t* pool_id, const uint64_t* ids, const uint64_t* scanned,
                       const uint32_t* q_item_off, const uint32_t* gthr, uint32_t nq, uint32_t k, uint64_t* out_ids,
                       float* out_dist, uint32_t* out_count, uint32_t* gkey, uint64_t* gtie, uint32_t pw,
                       cudaStream_t s) {
    (void)gkey;
    (void)gtie;
    (void)pw;
    cudaError_t e = launch_pdl(select_pool_kernel, dim3(nq), dim3(kPoolThreads), 0, s, pool_key, pool_id, ids, scanned,
                               q_item_off, gthr, k, out_ids, out_dist, out_count);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("CUDA launch failed (select_pool): ") + cudaGetErrorString(e));
        return PRAG_GPU_CUDA;
    }
    return PRAG_GPU_OK;
}

size_t select_smem_bytes() { return sizeof(SelShared); }

static int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("CUDA launch failed (") + what + "): " + cudaGetErrorString(e));
        return PRAG_GPU_CUDA;
    }
    return PRAG_GPU_OK;
}

int launch_coarse(const DeviceIndex& ix, const float* queries, uint32_t nq, float* out, cudaStream_t s) {
    if (ix.centroids4 != nullptr) {
        dim3 grid((ix.nlist + 127) / 128, (nq + 1) / 2);
        const size_t smem = size_t(2) * ix.d * sizeof(float);
        if (smem > 48 * 1024)
            PG_CUDA(ensure_smem(reinterpret_cast<const void*>(coarse_exact4_kernel), int(smem)));
        coarse_exact4_kernel<<<grid, 128, smem, s>>>(reinterpret_cast<const float4*>(ix.centroids4), queries, nq,
                                                     ix.nlist, ix.d, out);
        return check_launch("coarse4");
    }
    constexpr int QB = 8;
    dim3 grid((ix.nlist + 127) / 128, (nq + QB - 1) / QB);
    size_t smem = size_t(QB) * ix.d * sizeof(float);
    if (smem > 48 * 1024)
        PG_CUDA(ensure_smem(reinterpret_cast<const void*>(coarse_exact_kernel<QB>), int(smem)));
    coarse_exact_kernel<QB><<<grid, 128, smem, s>>>(ix.centroidsT, queries, nq, ix.nlist, ix.d, out);
    return check_launch("coarse");
}

static int set_sel_smem(const void* fn) {
    static_assert(sizeof(SelShared) < 227 * 1024, "selection smem");
    PG_CUDA(ensure_smem(reinterpret_cast<const void*>(fn), int(sizeof(SelShared))));
    return PRAG_GPU_OK;
}

int launch_select_probe(const DeviceIndex& ix, const float* coarse, uint32_t nq, uint32_t nprobe,
                        uint32_t* probe, float* probe_dist, uint32_t* gkey, uint64_t* gtie, cudaStream_t s) {
    PG_TRY(set_sel_smem(reinterpret_cast<const void*>(select_probe_kernel)));
    select_probe_kernel<<<nq, kSelThreads, sizeof(SelShared), s>>>(coarse, ix.nlist, nprobe, probe, probe_dist,
                                                                   gkey, gtie);
    return check_launch("select_probe");
}

int launch_plan(const DeviceIndex& ix, const SearchBuffers& b, cudaStream_t s) {
    plan_kernel<<<1, 1024, 0, s>>>(b.probe, ix.list_len, b.nq, b.nprobe, b.q_cand_off, b.out_scanned, b.items,
                                   b.num_items, b.item_cursor, b.item_cap);
    return check_launch("plan");
}

int launch_scan(const DeviceIndex& ix, const SearchBuffers& b, cudaStream_t s, int grid, float* glut) {
    const size_t lut_bytes = size_t(ix.nsq) * 256 * sizeof(float);
    const size_t res_bytes = ((ix.d + 3) & ~3u) * sizeof(float);
    const bool smem_lut = lut_bytes + res_bytes <= 200 * 1024;
    // no plain code array: read the lane-skewed tiles (m = 32 / 64)
    const bool skew = ix.codes == nullptr;
    const uint8_t* codes = skew ? ix.skew_codes : ix.codes;
#define PG_SCAN(SM, SK, SMEM, GL)                                                                               \
    do {                                                                                                       \
        PG_CUDA(ensure_smem(reinterpret_cast<const void*>(scan_kernel<SM, SK>), int(SMEM)));                  \
        scan_kernel<SM, SK><<<grid, 256, SMEM, s>>>(b.queries, ix.centroids, ix.codewordsT, ix.list_off,       \
                                                    ix.list_len, codes, ix.skew_off, ix.d, ix.nsq, ix.sub_dim, \
                                                    b.items, b.num_items, b.item_cursor, b.cand_dist,          \
                                                    b.cand_entry, GL);                                         \
    } while (0)
    if (smem_lut) {
        const size_t smem = lut_bytes + res_bytes;
        if (skew)
            PG_SCAN(true, true, smem, nullptr);
        else
            PG_SCAN(true, false, smem, nullptr);
    } else {
        const size_t smem = res_bytes;
        if (skew)
            PG_SCAN(false, true, smem, glut);
        else
            PG_SCAN(false, false, smem, glut);
    }
#undef PG_SCAN
    return check_launch("scan");
}

namespace {
// One thread per candidate of query blockIdx.y: the full-precision
// squared_l2(embeddings[chunk_id], query) of common.hpp:73-80, in the
// argument order of annindex.hpp:310 (diff = e - q), FMA-free.
__global__ void __launch_bounds__(256) rerank_kernel(const float* __restrict__ queries, uint32_t d,
                                                     const uint64_t* __restrict__ q_cand_off,
                                                     const uint32_t* __restrict__ cand_entry,
                                                     const uint64_t* __restrict__ ids, const float* __restrict__ emb,
                                                     float* __restrict__ cand_dist) {
    extern __shared__ float qs[];
    const uint32_t q = blockIdx.y;
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) qs[j] = queries[size_t(q) * d + j];
    __syncthreads();
    const uint64_t b0 = q_cand_off[q], b1 = q_cand_off[q + 1];
    const uint64_t o = b0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (o >= b1) return;
    const float* row = emb + size_t(ids[cand_entry[o]]) * d;
    float acc = 0.0f;
    if ((d & 3u) == 0) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
        for (uint32_t j4 = 0; j4 < d / 4; ++j4) {
            const float4 e = __ldg(r4 + j4);
            const float ev[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float diff = __fsub_rn(ev[t], qs[4 * j4 + t]);
                acc = __fadd_rn(acc, __fmul_rn(diff, diff));
            }
        }
    } else {
        for (uint32_t j = 0; j < d; ++j) {
            const float diff = __fsub_rn(__ldg(row + j), qs[j]);
            acc = __fadd_rn(acc, __fmul_rn(diff, diff));
        }
    }
    cand_dist[o] = acc;
}
}  // namespace

namespace {
// brute_force_search (annindex.hpp:244-257): the full-precision distance of
// every row, then the (distance, row id) top-k.
__global__ void __launch_bounds__(256) brute_dist_kernel(const float* __restrict__ emb, uint64_t n, uint32_t d,
                                                         const float* __restrict__ queries,
                                                         float* __restrict__ dist) {
    extern __shared__ float qs[];
    const uint32_t q = blockIdx.y;
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) qs[j] = queries[size_t(q) * d + j];
    __syncthreads();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* row = emb + i * d;
    float acc = 0.0f;
    for (uint32_t j = 0; j < d; ++j) {  // squared_l2(embeddings[i], query): diff = e - q
        const float diff = __fsub_rn(__ldg(row + j), qs[j]);
        acc = __fadd_rn(acc, __fmul_rn(diff, diff));
    }
    dist[size_t(q) * n + i] = acc;
}

struct RowSrc {
    const float* d;
    __device__ uint32_t key(uint32_t i) const { return ord_key(d[i]); }
    __device__ uint64_t tie(uint32_t i) const { return i; }
};

__global__ void __launch_bounds__(kSelThreads) brute_select_kernel(const float* __restrict__ dist, uint32_t n,
                                                                   uint32_t k, uint32_t* gkey, uint64_t* gtie,
                                                                   uint32_t pw, float* __restrict__ out_dist,
                                                                   uint64_t* __restrict__ out_ids,
                                                                   uint32_t* __restrict__ out_count) {
    extern __shared__ __align__(16) unsigned char smraw[];
    SelShared& sm = *reinterpret_cast<SelShared*>(smraw);
    const uint32_t q = blockIdx.x;
    block_topk(RowSrc{dist + size_t(q) * n}, n, k, sm, gkey + size_t(q) * pw, gtie + size_t(q) * pw,
               out_dist + size_t(q) * k, out_ids + size_t(q) * k, out_count + q);
}
}  // namespace

namespace {
__global__ void max_id_kernel(const uint64_t* __restrict__ ids, uint64_t n, unsigned long long* out) {
    unsigned long long m = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        if (ids[i] != ~0ull && ids[i] > m) m = ids[i];
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}
}  // namespace

// largest chunk id among the padded slots (padding slots hold ~0)
int max_chunk_id(const uint64_t* ids, uint64_t n, uint64_t* out) {
    unsigned long long* d = nullptr;
    PG_CUDA(cudaMalloc(&d, 8));
    cudaMemset(d, 0, 8);
    if (n) max_id_kernel<<<592, 256>>>(ids, n, d);
    unsigned long long h = 0;
    const cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    PG_CUDA(e);
    *out = h;
    return PRAG_GPU_OK;
}

int launch_brute_force(const float* emb, uint64_t n, uint32_t d, const float* queries, uint32_t nq, uint32_t k,
                       float* dist, uint32_t* gkey, uint64_t* gtie, uint32_t pw, uint64_t* out_ids, float* out_dist,
                       uint32_t* out_count, cudaStream_t s) {
    if (nq == 0) return PRAG_GPU_OK;
    brute_dist_kernel<<<dim3(uint32_t((n + 255) / 256), nq), 256, size_t(d) * 4, s>>>(emb, n, d, queries, dist);
    PG_TRY(check_launch("brute_dist"));
    PG_CUDA(ensure_smem(reinterpret_cast<const void*>(brute_select_kernel), int(sizeof(SelShared))));
    brute_select_kernel<<<nq, kSelThreads, sizeof(SelShared), s>>>(dist, uint32_t(n), k, gkey, gtie, pw, out_dist,
                                                                   out_ids, out_count);
    return check_launch("brute_select");
}

int launch_rerank(const DeviceIndex& ix, const SearchBuffers& b, const float* emb, uint64_t max_cand_q,
                  cudaStream_t s) {
    if (b.nq == 0 || max_cand_q == 0) return PRAG_GPU_OK;
    const uint64_t gx = (max_cand_q + 255) / 256;
    if (gx > 0x7fffffffull) {
        set_error("rerank: too many candidates per query");
        return PRAG_GPU_CONFIG;
    }
    rerank_kernel<<<dim3(uint32_t(gx), b.nq), 256, size_t(ix.d) * 4, s>>>(b.queries, ix.d, b.q_cand_off,
                                                                          b.cand_entry, ix.ids, emb, b.cand_dist);
    return check_launch("rerank");
}

int launch_final(const DeviceIndex& ix, const SearchBuffers& b, uint32_t* gkey, uint64_t* gtie, uint32_t pw,
                 cudaStream_t s) {
    PG_TRY(set_sel_smem(reinterpret_cast<const void*>(select_final_kernel)));
    select_final_kernel<<<b.nq, kSelThreads, sizeof(SelShared), s>>>(b.cand_dist, b.cand_entry, ix.ids,
                                                                      b.q_cand_off, b.k, b.out_ids, b.out_dist,
                                                                      b.out_count, gkey, gtie, pw);
    return check_launch("final");
}

int launch_merge(const uint64_t* ids, const float* dist, const uint32_t* count, const uint64_t* scanned,
                 uint32_t nparts, uint32_t nq, uint32_t kin, uint32_t k, uint64_t* out_ids, float* out_dist,
                 uint32_t* out_count, uint64_t* out_scanned, uint32_t* ckey, uint64_t* ctie, uint32_t* gkey,
                 uint64_t* gtie, uint32_t pw, cudaStream_t s) {
    PG_TRY(set_sel_smem(reinterpret_cast<const void*>(merge_kernel)));
    merge_kernel<<<nq, kSelThreads, sizeof(SelShared), s>>>(ids, dist, count, scanned, nparts, nq, kin, k, out_ids,
                                                             out_dist, out_count, out_scanned, ckey, ctie, gkey,
                                                             gtie, pw);
    return check_launch("merge");
}

uint32_t scan_chunk() { return kChunk; }
uint32_t sort_cap() { return kSortCap; }

}  // namespace pg
