// scan_skew.cu -- fast path of the list scan for PQ widths m = 32 and m = 64.
//
// Same arithmetic as annindex.hpp:285-305 (LUT entries and the ADC sum are
// sequential fp32 folds, FMA-free), laid out so the SMEM table gathers are
// bank-conflict free:
//
//  * Lane-skewed code tiles (HBM). A list is cut into tiles of 32 entries.
//    In round j lane t folds entry 32j+t, but starts it t steps late: at step
//    s it needs subquantizer (s - t) mod m -- entry 32j+t for s >= t, the
//    tail of entry 32(j-1)+t for s < t. The ingest stores, per tile and lane,
//    exactly the m code bytes lane t consumes in that round, in step order
//    ("skewed" tile, plus one tail tile per list). Lanes therefore always
//    touch 32 distinct subquantizers at the same step.
//  * Column-major LUT image (SMEM), [code][64] fp32 per 32 subquantizers,
//    with the wrap-around duplicated so lane t's column is s - t + 32: its
//    bank is (s - t) mod 32 -- distinct across the warp for every code value.
//    The address is PRMT(code byte, lane base) + a compile-time offset, one
//    instruction; the load is LDS [R + UR + imm].
//  * The lane-dependent switch between the finishing and the starting entry
//    is an FFMA with a 0/1 mask (x*1 + acc == acc + x and x*0 + acc == acc
//    exactly for finite x), so the fold order and every rounding are the
//    reference's.
//  * Each warp keeps an exact top-k (k <= 32) in registers, ordered by
//    (distance, chunk_id); a per-query threshold shared through global
//    memory (atomicMin on the k-th distance) prunes candidates; ids are
//    loaded only for candidates that pass.
#include <cstdint>
#include <utility>

#include "internal.h"

namespace pg {
namespace {

constexpr uint32_t kTileEntries = 32;
constexpr uint32_t kItemTiles = 512;  // tiles per scan work item (16384 entries)
constexpr uint32_t kLutPairs = 8;     // (query, list) pairs per LUT-kernel CTA

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// {c0, c1} = {a*b0 + c0, a*b1 + c1}: two independent IEEE fp32 FMAs (rn) in
// one FFMA2 with a scalar-broadcast first operand.
__device__ __forceinline__ void fma2_bcast(float& c0, float& c1, float a, float b0, float b1) {
    unsigned long long r;
    asm("{.reg .b64 A, B, C;\n"
        " mov.b64 A, {%1, %1};\n"
        " mov.b64 B, {%2, %3};\n"
        " mov.b64 C, {%4, %5};\n"
        " fma.rn.f32x2 %0, A, B, C;}"
        : "=l"(r)
        : "f"(a), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
    c0 = __uint_as_float(uint32_t(r));
    c1 = __uint_as_float(uint32_t(r >> 32));
}

__device__ __forceinline__ uint32_t ord_key(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// ----------------------------------------------------------- LUT images
// {r0 - w, r1 - w}: one FADD2 with a scalar-broadcast operand; a subtraction
// is a single rounding, identical to two __fsub_rn. (Packed MUL/ADD pairs are
// NOT used anywhere: ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2,
// which would change the reference's rounding.)
__device__ __forceinline__ void sub2_bcast(float r0, float r1, float w, float& d0, float& d1) {
    unsigned long long out;
    asm("{.reg .b64 A, B;\n"
        " mov.b64 A, {%1, %2};\n"
        " mov.b64 B, {%3, %3};\n"
        " sub.rn.f32x2 %0, A, B;}"
        : "=l"(out)
        : "f"(r0), "f"(r1), "f"(w));
    d0 = __uint_as_float(uint32_t(out));
    d1 = __uint_as_float(uint32_t(out >> 32));
}

// Grid: (ceil(npairs / kLutPairs), m / 8). CTA: 256 threads = 256 codes; it
// computes subquantizers [8*blockIdx.y, +8) of T[sq][code] =
// squared_l2(r_sq, w[sq][code], sub_dim) (annindex.hpp:292-297, residual
// r = q - c_list) for kLutPairs pairs and writes the compact table
// luts[pair][sq][256] (coalesced; the scan CTA expands it into its SMEM
// image). Residuals sit in SMEM as [sq][j][pair] so one LDS.128 broadcasts
// four pairs' values.
template <int M, int SUBC>  // SUBC: compile-time sub_dim (0 = runtime `sub`, <= 16)
__global__ void __launch_bounds__(256, 2) lut_kernel(const float* __restrict__ queries,
                                                     const float* __restrict__ centroids,
                                                     const float* __restrict__ codewords,
                                                     const uint32_t* __restrict__ probe,
                                                     const uint32_t* __restrict__ list_len, uint32_t nq,
                                                     uint32_t nprobe, uint32_t d, uint32_t sub,
                                                     float* __restrict__ luts) {
    constexpr int P = kLutPairs;  // 8
    constexpr int JMAX = SUBC ? SUBC : 16;
    if (SUBC) sub = SUBC;
    __shared__ __align__(16) float resid[8 * 16 * P];  // [sq_local][j][pair]
    __shared__ uint32_t s_q[P], s_list[P];
    const uint32_t npairs = nq * nprobe;
    const uint32_t p0 = blockIdx.x * P;
    const uint32_t sq0 = blockIdx.y * 8;
    if (threadIdx.x < P) {
        const uint32_t pair = p0 + threadIdx.x;
        uint32_t list = 0xffffffffu;
        if (pair < npairs) {
            list = probe[pair];
            if (list_len[list] == 0) list = 0xffffffffu;
        }
        s_q[threadIdx.x] = pair / nprobe;
        s_list[threadIdx.x] = list;
    }
    __syncthreads();
    uint32_t live = 0;  // bitmask of pairs with a non-empty list
#pragma unroll
    for (int p = 0; p < P; ++p) live |= (s_list[p] != 0xffffffffu) << p;
    if (!live) return;
    // residual r = q - c_list (annindex.hpp:292) for this CTA's 8 subquantizers
    const uint32_t span = 8 * sub;  // contiguous dims [sq0*sub, +span)
    for (uint32_t t = threadIdx.x; t < span * P; t += blockDim.x) {
        const uint32_t p = t / span, k = t - p * span;
        const uint32_t sl = k / sub, j = k - sl * sub;
        float v = 0.0f;
        if (s_list[p] != 0xffffffffu) {
            const uint32_t dim = sq0 * sub + k;
            v = __fsub_rn(queries[size_t(s_q[p]) * d + dim], centroids[size_t(s_list[p]) * d + dim]);
        }
        resid[(sl * 16 + j) * P + p] = v;
    }
    __syncthreads();
    const uint32_t code = threadIdx.x;
#pragma unroll 1
    for (uint32_t i = 0; i < 8; ++i) {
        const uint32_t sq = sq0 + i;
        float w[JMAX];
        const float* wp = codewords + (size_t(sq) * 256 + code) * sub;
#pragma unroll
        for (int j = 0; j < JMAX; ++j)
            if (j < int(sub)) w[j] = __ldg(wp + j);
        float acc[P];
#pragma unroll
        for (int p = 0; p < P; ++p) acc[p] = 0.0f;
        const float* rr = resid + (i * 16) * P;
#pragma unroll
        for (int j = 0; j < JMAX; ++j) {
            if (j < int(sub)) {
                const float4 ra = *reinterpret_cast<const float4*>(rr + j * P);
                const float4 rb = *reinterpret_cast<const float4*>(rr + j * P + 4);
                float dd[P];
                sub2_bcast(ra.x, ra.y, w[j], dd[0], dd[1]);
                sub2_bcast(ra.z, ra.w, w[j], dd[2], dd[3]);
                sub2_bcast(rb.x, rb.y, w[j], dd[4], dd[5]);
                sub2_bcast(rb.z, rb.w, w[j], dd[6], dd[7]);
#pragma unroll
                for (int p = 0; p < P; ++p) acc[p] = __fadd_rn(acc[p], __fmul_rn(dd[p], dd[p]));
            }
        }
#pragma unroll
        for (int p = 0; p < P; ++p)
            if (live >> p & 1u) luts[(size_t(p0 + p) * M + sq) * 256 + code] = acc[p];
    }
}

// ------------------------------------------------------------------- scan
template <int M>
struct SkewCfg;
template <>
struct SkewCfg<32> {
    static constexpr int kWarps = 8;      // 2 CTAs per SM
    static constexpr int kDepth = 4;      // code tiles in flight per warp (TMA ring, power of 2)
    static constexpr int kMinBlocks = 2;
};
template <>
struct SkewCfg<64> {
    static constexpr int kWarps = 16;     // 1 CTA per SM (128 KB LUT image)
    static constexpr int kDepth = 2;
    static constexpr int kMinBlocks = 1;
};

template <int M>
constexpr size_t skew_smem_bytes() {
    return size_t(M / 32) * 65536 + size_t(SkewCfg<M>::kWarps) * SkewCfg<M>::kDepth * 32 * M +
           8 * (1 + SkewCfg<M>::kWarps * SkewCfg<M>::kDepth) + 32;
}

// LUT gather: 32-bit shared::cta address (uniform base folded by ptxas into
// LDS [R + UR + imm]) plus a compile-time offset.
template <int IMM>
__device__ __forceinline__ float lds_lut(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(IMM));
    return v;
}

__device__ __forceinline__ uint4 lds_u4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

// One step of the skewed fold: lane's code byte S -> table column, gather,
// and the masked {cur, prev} update (steps >= 32 always belong to `cur`).
template <int M, int S>
__device__ __forceinline__ void skew_step(const uint32_t* w, uint32_t bt, uint32_t lutb, float& cur, float& prev,
                                          const float* mk, const float* nk) {
    constexpr int r = S >> 5;
    const uint32_t addr = __byte_perm(w[S >> 2], bt, 0x7604u | (uint32_t(S & 3) << 4)) + lutb;
    const float t = lds_lut<r * 65536 + (S - 32 * r) * 4>(addr);
    if constexpr (S < 32) {
        fma2_bcast(cur, prev, t, mk[S], nk[S]);
    } else {
        cur = __fadd_rn(cur, t);
    }
}

template <int M, int... S>
__device__ __forceinline__ void skew_round(const uint32_t* w, uint32_t bt, uint32_t lutb, float& cur, float& prev,
                                           const float* mk, const float* nk, std::integer_sequence<int, S...>) {
    (skew_step<M, S>(w, bt, lutb, cur, prev, mk, nk), ...);
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

struct WarpTopK {
    uint32_t key;  // raw float bits of the distance (distances are >= +0)
    uint64_t id;
};

// Persistent CTAs pull work items {pair, tile_begin, tile_end} (largest
// first). Per item: TMA bulk-copy the pair's LUT image into SMEM; each warp
// scans a contiguous tile range, its code tiles streamed through a per-warp
// ring of kDepth TMA bulk copies (one elected lane, one mbarrier per slot).
template <int M>
__global__ void __launch_bounds__(SkewCfg<M>::kWarps * 32, SkewCfg<M>::kMinBlocks)
    scan_skew_kernel(const uint4* __restrict__ items, const uint32_t* __restrict__ num_items,
                     uint32_t* __restrict__ cursor, const uint32_t* __restrict__ probe,
                     const uint32_t* __restrict__ list_len, const uint64_t* __restrict__ skew_off,
                     const uint8_t* __restrict__ skew_codes, const uint64_t* __restrict__ list_off,
                     const uint64_t* __restrict__ ids, const float* __restrict__ luts, uint32_t nprobe,
                     uint32_t k, uint32_t* __restrict__ gthr, const uint32_t* __restrict__ q_item_off,
                     uint32_t* __restrict__ pool_cnt, uint32_t* __restrict__ pool_key,
                     uint64_t* __restrict__ pool_id) {
    constexpr int R = M / 32;
    constexpr int kWarps = SkewCfg<M>::kWarps;
    constexpr int D = SkewCfg<M>::kDepth;
    constexpr int kChunks = M / 16;              // uint4 per lane per round
    constexpr uint32_t kTileBytes = 32u * M;     // bytes per tile
    constexpr uint32_t kImgBytes = R * 65536u;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* ring = smem + kImgBytes;                                   // [warps][D][tile]
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + size_t(kWarps) * D * kTileBytes);  // [0]=LUT
    uint32_t* s_item = reinterpret_cast<uint32_t*>(bars + 1 + kWarps * D);
    uint32_t* s_thr = s_item + 1;  // the CTA's view of the query threshold

    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t bt = (32u - lane) * 4u;  // lane's column offset (bytes), byte 0 of the address
    const uint32_t lut_s = smem_u32(smem);  // shared::cta address of the LUT image
    unsigned char* wring = ring + size_t(warp) * D * kTileBytes;
    uint64_t* wbar = bars + 1 + warp * D;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 1 + kWarps * D; ++i) mbar_init(bars + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t total = *num_items;
    uint32_t consumed = 0;  // tiles this warp has taken from its ring (slot/parity bookkeeping)
    // step masks: {1, 0} where step s >= lane (the starting entry), {0, 1}
    // before (the finishing entry); one FFMA2 updates {cur, prev}.
    float mk[32], nk[32];
#pragma unroll
    for (int s = 0; s < 32; ++s) {
        mk[s] = (uint32_t(s) >= lane) ? 1.0f : 0.0f;
        nk[s] = (uint32_t(s) >= lane) ? 0.0f : 1.0f;
    }

    uint32_t prev_q = 0xffffffffu;
    for (;;) {
        __syncthreads();  // every warp is done with the previous item (LUT image, s_thr)
        if (threadIdx.x == 0) {
            if (prev_q != 0xffffffffu) atomicMin(gthr + prev_q, *s_thr);  // publish to other CTAs
            const uint32_t nx = atomicAdd(cursor, 1u);
            *s_item = nx;
            if (nx < total) *s_thr = ld_relaxed(gthr + items[nx].x / nprobe);
        }
        __syncthreads();
        const uint32_t it = *s_item;
        if (it >= total) break;
        const uint4 w4 = items[it];
        const uint32_t pair = w4.x, tb = w4.y, te = w4.z;
        const uint32_t q = pair / nprobe;
        prev_q = q;
        const uint32_t list = probe[pair];
        const uint32_t len = list_len[list];
        // expand the pair's compact table T[sq][256] (L2) into the SMEM image:
        // lane = subquantizer (bank = column mod 32 = sq: conflict-free STS),
        // warps stride over groups of 4 codes (one LDG.128 each)
        {
            const float4* src = reinterpret_cast<const float4*>(luts + size_t(pair) * M * 256);
            float* img = reinterpret_cast<float*>(smem);
#pragma unroll 1
            for (uint32_t sqb = 0; sqb < uint32_t(M); sqb += 32) {
                const uint32_t sq = sqb + lane;
#pragma unroll 4
                for (uint32_t g = warp; g < 64; g += kWarps) {
                    const float4 v = src[sq * 64 + g];
                    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        float* row = img + (g * 4 + i) * 64;
                        // table 0: cur column sq + 32 (sq < 32), finishing column sq - (m - 32)
                        if (sq < 32) row[32 + sq] = vv[i];
                        if (sq + 32 >= uint32_t(M)) row[sq + 32 - M] = vv[i];
#pragma unroll
                        for (int r_ = 1; r_ < R; ++r_) {
                            const int c = int(sq) - 32 * (r_ - 1);
                            if (c >= 0 && c <= 63) row[r_ * 16384 + c] = vv[i];
                        }
                    }
                }
            }
        }
        // this warp's share of tiles [tb, te); it also reads tile b (the tail
        // of its last entries), so it streams b - a + 1 tiles
        const uint32_t ntile = te - tb;
        const uint32_t per = (ntile + kWarps - 1) / kWarps;
        const uint32_t a = tb + warp * per;
        const uint32_t b = min(te, a + per);
        const unsigned char* tiles = skew_codes + skew_off[list] * kTileBytes;
        const uint64_t lbase = list_off[list];
        if (a < b && lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (uint32_t i = 0; i < uint32_t(D) && a + i <= b; ++i) {
                const uint32_t slot = (consumed + i) % D;
                mbar_expect_tx(wbar + slot, kTileBytes);
                bulk_g2s(wring + slot * kTileBytes, tiles + size_t(a + i) * kTileBytes, kTileBytes, wbar + slot);
            }
        }
        __syncthreads();  // SMEM image complete
        if (a >= b) continue;

        WarpTopK tk{0xffffffffu, ~0ull};
        uint32_t thr_key = 0xffffffffu;
        uint32_t g_thr = *reinterpret_cast<volatile uint32_t*>(s_thr);
        float cur = 0.0f, prev = 0.0f;
        const uint32_t ring_s = smem_u32(wring);
        for (uint32_t j = a; j <= b; ++j, ++consumed) {
            const uint32_t slot = consumed % D;
            mbar_wait(wbar + slot, (consumed / D) & 1u);
            uint32_t wd[M / 4];
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
                const uint4 v = lds_u4(ring_s + slot * kTileBytes + c * 512 + lane * 16);
                wd[4 * c] = v.x;
                wd[4 * c + 1] = v.y;
                wd[4 * c + 2] = v.z;
                wd[4 * c + 3] = v.w;
            }
            const uint32_t g_cta = *reinterpret_cast<volatile uint32_t*>(s_thr);  // used after the steps
            skew_round<M>(wd, bt, lut_s, cur, prev, mk, nk, std::make_integer_sequence<int, M>{});
            // the codes of this slot are consumed (every lane's LDS.128 result
            // was used by the steps above): refill it with tile j + D
            __syncwarp();
            if (lane == 0 && j + D <= b) {
                mbar_expect_tx(wbar + slot, kTileBytes);
                bulk_g2s(wring + slot * kTileBytes, tiles + size_t(j + D) * kTileBytes, kTileBytes, wbar + slot);
            }
            g_thr = min(g_thr, g_cta);
            // entry 32(j-1)+lane is complete in `prev`
            const uint32_t e = (j - 1) * kTileEntries + lane;
            const bool valid = j > a && e < len;
            const uint32_t key = __float_as_uint(prev);
            prev = cur;
            cur = 0.0f;
            const uint32_t lim = min(thr_key, g_thr);
            bool pass = valid && key <= lim;
            unsigned bal = __ballot_sync(0xffffffffu, pass);
            if (bal) {
                const uint64_t myid = pass ? ids[lbase + e] : 0ull;
                while (bal) {
                    const int src = __ffs(bal) - 1;
                    bal &= bal - 1;
                    const uint32_t ck = __shfl_sync(0xffffffffu, key, src);
                    const uint64_t ci = __shfl_sync(0xffffffffu, myid, src);
                    if (ck > thr_key) continue;  // threshold tightened by an earlier insertion
                    // lanes whose element sorts after the candidate
                    const bool gt = tk.key > ck || (tk.key == ck && tk.id > ci);
                    const unsigned gm = __ballot_sync(0xffffffffu, gt);
                    const int pos = gm ? __ffs(gm) - 1 : 32;
                    if (pos < int(k)) {
                        const uint32_t uk = __shfl_up_sync(0xffffffffu, tk.key, 1);
                        const uint64_t ui = __shfl_up_sync(0xffffffffu, tk.id, 1);
                        if (int(lane) > pos) {
                            tk.key = uk;
                            tk.id = ui;
                        } else if (int(lane) == pos) {
                            tk.key = ck;
                            tk.id = ci;
                        }
                        thr_key = __shfl_sync(0xffffffffu, tk.key, k - 1);
                    }
                }
                if (thr_key < g_thr) {
                    if (lane == 0) atomicMin(s_thr, thr_key);
                    g_thr = thr_key;
                }
            }
        }
        // publish this warp's list into the query's candidate pool
        const unsigned have = __ballot_sync(0xffffffffu, lane < k && tk.key != 0xffffffffu);
        const uint32_t cnt = __popc(have);
        if (cnt) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(pool_cnt + q, cnt);
            base = __shfl_sync(0xffffffffu, base, 0);
            const size_t poff = size_t(q_item_off[q]) * kWarps * k;
            if (lane < cnt) {
                pool_key[poff + base + lane] = ord_key(__uint_as_float(tk.key));
                pool_id[poff + base + lane] = tk.id;
            }
        }
    }
}

// Work items for the fast path: per (q, p) pair, ceil(len/32) tiles cut into
// items of <= kItemTiles tiles, emitted largest-first (log2 size buckets) so
// the big lists set each query's threshold early and the small ones fill the
// tail. q_item_off[q] = prefix of per-query item counts (candidate-pool
// offsets). Also resets the per-query threshold and pool counters.
__global__ void __launch_bounds__(1024) plan_skew_kernel(const uint32_t* __restrict__ probe,
                                                         const uint32_t* __restrict__ list_len, uint32_t nq,
                                                         uint32_t nprobe, uint64_t* __restrict__ scanned,
                                                         uint4* __restrict__ items, uint32_t* __restrict__ num_items,
                                                         uint32_t* __restrict__ cursor, uint32_t* __restrict__ q_item_off,
                                                         uint32_t* __restrict__ gthr, uint32_t* __restrict__ pool_cnt,
                                                         uint64_t item_cap) {
    __shared__ uint32_t tmp[33];
    __shared__ uint32_t bucket_cnt[32], bucket_pos[32];
    const uint32_t P = nq * nprobe;
    if (threadIdx.x < 32) bucket_cnt[threadIdx.x] = 0;
    __syncthreads();
    // pass 1: per-query item counts (prefix) and bucket histogram
    uint32_t carry = 0;
    for (uint32_t base = 0; base < P; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const bool valid = i < P;
        const uint32_t len = valid ? list_len[probe[i]] : 0;
        const uint32_t tiles = (len + kTileEntries - 1) / kTileEntries;
        const uint32_t nit = (tiles + kItemTiles - 1) / kItemTiles;
        for (uint32_t j = 0; j < nit; ++j) {
            const uint32_t t = min(tiles, (j + 1) * kItemTiles) - j * kItemTiles;
            atomicAdd(&bucket_cnt[31 - __clz(t)], 1u);
        }
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        uint32_t incl = nit;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) tmp[w] = incl;
        __syncthreads();
        if (w == 0) {
            const int nw = blockDim.x >> 5;
            uint32_t x = lane < nw ? tmp[lane] : 0u, xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t t = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += t;
            }
            if (lane < nw) tmp[lane] = xi - x;
            if (lane == nw - 1) tmp[32] = xi;
        }
        __syncthreads();
        const uint32_t excl = carry + tmp[w] + incl - nit;
        if (valid && i % nprobe == 0) q_item_off[i / nprobe] = excl;
        carry += tmp[32];
        __syncthreads();
    }
    // bucket start positions, largest bucket first
    if (threadIdx.x == 0) {
        uint32_t pos = 0;
        for (int bkt = 31; bkt >= 0; --bkt) {
            bucket_pos[bkt] = pos;
            pos += bucket_cnt[bkt];
        }
    }
    __syncthreads();
    // pass 2: scatter items
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        const uint32_t len = list_len[probe[i]];
        const uint32_t tiles = (len + kTileEntries - 1) / kTileEntries;
        const uint32_t nit = (tiles + kItemTiles - 1) / kItemTiles;
        for (uint32_t j = 0; j < nit; ++j) {
            const uint32_t te = min(tiles, (j + 1) * kItemTiles);
            const uint32_t slot = atomicAdd(&bucket_pos[31 - __clz(te - j * kItemTiles)], 1u);
            if (slot < item_cap) items[slot] = make_uint4(i, j * kItemTiles, te, 0u);
        }
    }
    if (threadIdx.x == 0) {
        *num_items = carry;
        *cursor = 0;
        q_item_off[nq] = carry;
    }
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
        gthr[q] = 0xffffffffu;
        pool_cnt[q] = 0;
        uint64_t s = 0;
        for (uint32_t p = 0; p < nprobe; ++p) s += list_len[probe[q * nprobe + p]];
        scanned[q] = s;
    }
}

}  // namespace

uint32_t skew_item_tiles() { return kItemTiles; }
uint32_t skew_warps(uint32_t m) { return m == 32 ? SkewCfg<32>::kWarps : SkewCfg<64>::kWarps; }
uint32_t skew_ctas_per_sm(uint32_t m) { return m == 32 ? 2 : 1; }

static int check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("CUDA launch failed (") + what + "): " + cudaGetErrorString(e));
        return PRAG_GPU_CUDA;
    }
    return PRAG_GPU_OK;
}

int launch_plan_skew(const DeviceIndex& ix, const uint32_t* probe, uint32_t nq, uint32_t nprobe,
                     uint64_t* scanned, uint4* items, uint32_t* num_items, uint32_t* cursor, uint32_t* q_item_off,
                     uint32_t* gthr, uint32_t* pool_cnt, uint64_t item_cap, cudaStream_t s) {
    plan_skew_kernel<<<1, 1024, 0, s>>>(probe, ix.list_len, nq, nprobe, scanned, items, num_items, cursor,
                                        q_item_off, gthr, pool_cnt, item_cap);
    return check("plan_skew");
}

int launch_lut_images(const DeviceIndex& ix, const float* queries, const uint32_t* probe, uint32_t nq,
                      uint32_t nprobe, float* luts, cudaStream_t s) {
    const uint32_t npairs = nq * nprobe;
    dim3 grid((npairs + kLutPairs - 1) / kLutPairs, ix.nsq / 8);
#define PG_LUT(MM, SS)                                                                             \
    lut_kernel<MM, SS><<<grid, 256, 0, s>>>(queries, ix.centroids, ix.codewords, probe, ix.list_len, nq, \
                                            nprobe, ix.d, ix.sub_dim, luts)
    if (ix.nsq == 32 && ix.sub_dim == 12)
        PG_LUT(32, 12);
    else if (ix.nsq == 32)
        PG_LUT(32, 0);
    else if (ix.sub_dim == 6)
        PG_LUT(64, 6);
    else
        PG_LUT(64, 0);
#undef PG_LUT
    return check("lut_images");
}

int launch_scan_skew(const DeviceIndex& ix, const uint4* items, const uint32_t* num_items, uint32_t* cursor,
                     const uint32_t* probe, const float* images, uint32_t nprobe, uint32_t k, uint32_t* gthr,
                     const uint32_t* q_item_off, uint32_t* pool_cnt, uint32_t* pool_key, uint64_t* pool_id,
                     int grid, cudaStream_t s) {
    if (ix.nsq == 32) {
        const size_t smem = skew_smem_bytes<32>();
        PG_CUDA(cudaFuncSetAttribute(scan_skew_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        PG_CUDA(cudaFuncSetAttribute(scan_skew_kernel<32>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        scan_skew_kernel<32><<<grid, SkewCfg<32>::kWarps * 32, smem, s>>>(
            items, num_items, cursor, probe, ix.list_len, ix.skew_off, ix.skew_codes, ix.list_off, ix.ids, images,
            nprobe, k, gthr, q_item_off, pool_cnt, pool_key, pool_id);
    } else {
        const size_t smem = skew_smem_bytes<64>();
        PG_CUDA(cudaFuncSetAttribute(scan_skew_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        PG_CUDA(cudaFuncSetAttribute(scan_skew_kernel<64>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        scan_skew_kernel<64><<<grid, SkewCfg<64>::kWarps * 32, smem, s>>>(
            items, num_items, cursor, probe, ix.list_len, ix.skew_off, ix.skew_codes, ix.list_off, ix.ids, images,
            nprobe, k, gthr, q_item_off, pool_cnt, pool_key, pool_id);
    }
    return check("scan_skew");
}

// Host-side construction of the lane-skewed tile layout from list-major
// codes (see the file comment). out must hold skew_off[nlist] tiles.
void build_skew_layout(const HostIndex& h, uint32_t m, std::vector<uint64_t>& skew_off,
                       std::vector<uint8_t>& out) {
    const uint32_t nl = h.nlist;
    skew_off.assign(size_t(nl) + 1, 0);
    for (uint32_t l = 0; l < nl; ++l) {
        const uint64_t len = h.list_off[l + 1] - h.list_off[l];
        const uint64_t tiles = len ? (len + 31) / 32 + 1 : 0;
        skew_off[l + 1] = skew_off[l] + tiles;
    }
    const size_t tile_bytes = size_t(32) * m;
    out.assign(skew_off[nl] * tile_bytes, 0);
    for (uint32_t l = 0; l < nl; ++l) {
        const uint64_t len = h.list_off[l + 1] - h.list_off[l];
        if (!len) continue;
        const uint8_t* codes = h.codes.data() + h.list_off[l] * m;
        const uint64_t tiles = skew_off[l + 1] - skew_off[l];
        for (uint64_t j = 0; j < tiles; ++j) {
            uint8_t* tile = out.data() + (skew_off[l] + j) * tile_bytes;
            for (uint32_t t = 0; t < 32; ++t) {
                for (uint32_t s = 0; s < m; ++s) {
                    uint64_t e;
                    uint32_t byte;
                    bool ok;
                    if (s >= t) {
                        e = j * 32 + t;
                        byte = s - t;
                        ok = e < len;
                    } else {
                        ok = j >= 1;
                        e = (j - 1) * 32 + t;
                        byte = s - t + m;
                        ok = ok && e < len;
                    }
                    // lane t's byte s lives in 16-byte chunk s/16 at chunk*512 + t*16 + s%16
                    tile[(s / 16) * 512 + t * 16 + (s % 16)] = ok ? codes[e * m + byte] : 0;
                }
            }
        }
    }
}

}  // namespace pg
