// coarse_tc.cu -- K1 on the tensor cores: the coarse quantizer
// (annindex.hpp:277-281) as a tcgen05 GEMM pre-filter plus an exact rescoring
// of the boundary window.
//
// The reference orders lists by squared_l2(q, c) (common.hpp:73-80), a
// sequential fp32 fold; a GEMM-form ||q||^2 + ||c||^2 - 2 q.c cannot reproduce
// it bit for bit, and a near-tie at the nprobe-th list would swap a whole
// probed list. So:
//
//  K1  coarse_tc_kernel     S = C . Q^T with 3xTF32 (hi*hi + hi*lo + lo*hi,
//                           kind::tf32, fp32 accumulate in TMEM), one CTA per
//                           128 centroids x <= 256 queries. Epilogue: the
//                           approximate distance A = ||q||^2 + ||c||^2 - 2 S and
//                           a rigorous bound E >= |A - R| (R = the reference's
//                           exact value), written as (A + E, A - E).
//  K1b select_window_kernel per query: U = nprobe-th smallest (A + E); every
//                           list of the true top-nprobe has A - E <= R <= U, so
//                           the window {c : A - E <= U} holds them all (and
//                           anything outside it is strictly worse). The window
//                           is rescored with the exact FMA-free fold and
//                           ranked by (R, list id) -> probe[q][0..nprobe).
//
// Error bound (E = kBoundC(d) * (||q||^2 + ||c||^2)): split inputs x = hi + lo
// (hi = x with the low 13 mantissa bits cleared, exact; lo = x - hi, exact,
// truncated to tf32 by the MMA: error < 2^-20 |x|); dropped lo*lo and
// truncation terms < 3 * 2^-20 |q_j c_j|; fp32 accumulation of d terms in any
// order and with truncation < d * 2^-23 sum |q_j c_j|; sum |q_j c_j| <=
// (||q||^2 + ||c||^2) / 2; the norms' own error < d * 2^-24 each; and the
// reference fold R itself is within (d + 3) * 2^-24 * D of the real distance
// D <= 2 (||q||^2 + ||c||^2). The sum of these is < (6d + 64) * 2^-24; K1
// uses (8d + 256) * 2^-24 (~1.7x margin at d = 384), and the GPU parity suite
// checks the observed |A - R| against it.
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace pg {
namespace {

constexpr uint32_t kTcRows = 128;   // centroids per CTA (MMA M)
constexpr uint32_t kTcKBlock = 32;  // K elements per pipeline stage
constexpr uint32_t kTcMaxN = 64;    // queries per CTA (MMA N)
constexpr uint32_t kTcSliceBlocks = 3;  // K blocks per CTA (K slice of 96)
constexpr uint32_t kTcMaxSlices = 8;    // d <= 8 * 96 on the tensor-core path

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TC_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra TC_WAIT;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase), "r"(0x989680u)
        : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8 rows
// x 16 B; `lbo` = byte stride between the two K-adjacent core matrices of one
// MMA (K = 8 tf32), `sbo` = byte stride between 8-row groups.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((saddr & 0x3ffffu) >> 4) | (uint64_t(lbo >> 4) << 16) | (uint64_t(sbo >> 4) << 32) |
           (uint64_t(1) << 46);  // version 1 (sm_100), base offset 0, layout SWIZZLE_NONE
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// K1. Grid (nlist / 128, ceil(nq / N), ceil(d / 96)); 128 threads. A CTA
// owns 128 centroids x N queries x one 96-wide K slice (3 blocks of 32), so
// nlist = 4096, d = 384 runs 128 CTAs. The centroid blocks (cent_tc, 16 KiB
// of fp32 each, split into hi | lo in SMEM after they land) are bulk-copied
// on one mbarrier before waiting on the previous kernel; the query rows of the slice are read by all threads
// (one float4 per lane, four rows in flight per warp) and split hi/lo straight
// into the core-matrix layout; 36 MMAs are issued by one thread, and the
// partial dot products go out as partial[slice][q][c] (summed, with the norms
// and the bound, by K1b).
__global__ void __launch_bounds__(128, 1) coarse_tc_kernel(const float* __restrict__ cent_tc,
                                                           const float* __restrict__ queries, uint32_t nq,
                                                           uint32_t nlist, uint32_t d, uint32_t n_tile,
                                                           float* __restrict__ partial) {
    CT_BEGIN;
    // let K1b's CTAs launch onto free SMs now (griddepcontrol.wait in K1b
    // still waits for this whole grid and its memory)
    pdl_trigger();
    extern __shared__ __align__(1024) unsigned char sm[];
    const uint32_t N = n_tile;                                // multiple of 8, <= kTcMaxN
    const uint32_t kA = 2 * kTcRows * kTcKBlock * 4;          // one K block of A, hi + lo: 32 KiB
    const uint32_t kBp = N * kTcKBlock * 4;                   // one part of one K block of B
    const uint32_t nkb_all = d / kTcKBlock;
    const uint32_t kb0 = blockIdx.z * kTcSliceBlocks;
    const uint32_t nkb = min(kTcSliceBlocks, nkb_all - kb0);
    unsigned char* sA = sm;                                   // [nkb][hi | lo]
    unsigned char* sB = sA + kTcSliceBlocks * kA;             // [nkb][hi | lo][kBp]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kTcSliceBlocks * 2 * kBp);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t tile = blockIdx.x, q0 = blockIdx.y * N;
    const uint32_t nvalid = min(N, nq - q0);
    uint32_t ncols = 32;
    while (ncols < N) ncols <<= 1;

    if (tid == 0) {
        bar_init(bars, 1);
        bar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        bar_expect_tx(bars, nkb * (kA / 2));
        // index data: it does not depend on the previous kernel. Only the fp32
        // centroids travel (half the bytes of a pre-split hi | lo copy); they
        // land in the hi slot and are split in SMEM below.
        for (uint32_t i = 0; i < nkb; ++i)
            bulk_load(sA + i * kA, cent_tc + (size_t(tile) * nkb_all + kb0 + i) * (kTcRows * kTcKBlock), kA / 2,
                      bars);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    pdl_wait();
    CT_WAITED(0);
    // B: element (n, k) of a part at (k/4) * (N * 16) + (n/8) * 128 + (n%8) * 16 + (k%4) * 4,
    // so the 4 consecutive k of one float4 are one 16-byte store. Lane = float4
    // of the row (nkb * 8 <= 24 lanes busy), warp w takes rows w, w + 4, ...
    const uint32_t k4n = nkb * (kTcKBlock / 4);
    if (lane < k4n) {
        const uint32_t k = lane * 4, blk = k / kTcKBlock, kk = k % kTcKBlock;
        unsigned char* b = sB + blk * 2 * kBp + (kk >> 2) * (N * 16);
        const float* qbase = queries + size_t(kb0) * kTcKBlock + k;
        const bool vec = (reinterpret_cast<uintptr_t>(queries) & 15u) == 0;  // d % 32 == 0: rows stay aligned
        // all of the warp's rows (N / 4 <= 16) in flight at once
        constexpr uint32_t R = kTcMaxN / 4;
        float4 x[R];
#pragma unroll
        for (uint32_t u = 0; u < R; ++u) {
            const uint32_t n = warp + 4 * u;
            x[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (n < nvalid) {
                const float* src = qbase + size_t(q0 + n) * d;
                x[u] = vec ? *reinterpret_cast<const float4*>(src) : make_float4(src[0], src[1], src[2], src[3]);
            }
        }
#pragma unroll
        for (uint32_t u = 0; u < R; ++u) {
            const uint32_t n = warp + 4 * u;
            if (n < N) {
                const float4 hi = make_float4(tf32_hi(x[u].x), tf32_hi(x[u].y), tf32_hi(x[u].z), tf32_hi(x[u].w));
                const float4 lo = make_float4(__fsub_rn(x[u].x, hi.x), __fsub_rn(x[u].y, hi.y),
                                              __fsub_rn(x[u].z, hi.z), __fsub_rn(x[u].w, hi.w));
                const uint32_t off = (n >> 3) * 128 + (n & 7) * 16;
                *reinterpret_cast<float4*>(b + off) = hi;
                *reinterpret_cast<float4*>(b + kBp + off) = lo;
            }
        }
    }
    __syncthreads();  // the barriers' init is visible to every thread
    // A: split the staged centroids x into hi = x with the low 13 mantissa
    // bits cleared and lo = x - hi (exact), element-wise in place: the same
    // operands the round-1 host-side pre-split produced
    bar_wait(bars, 0);
    for (uint32_t i = 0; i < nkb; ++i) {
        float4* hp = reinterpret_cast<float4*>(sA + i * kA);
        float4* lp = reinterpret_cast<float4*>(sA + i * kA + kA / 2);
        for (uint32_t e = tid; e < kTcRows * kTcKBlock / 4; e += 128) {
            const float4 x = hp[e];
            const float4 hi = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
            hp[e] = hi;
            lp[e] = make_float4(__fsub_rn(x.x, hi.x), __fsub_rn(x.y, hi.y), __fsub_rn(x.z, hi.z), __fsub_rn(x.w, hi.w));
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic STS -> tensor-core reads
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    CT_MARK(6);
    const uint32_t tmem = *tmem_slot;
    if (tid == 0) {
        bar_wait(bars, 0);
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((kTcRows >> 4) << 24);
        for (uint32_t i = 0; i < nkb; ++i) {
            const uint32_t a0 = smem_addr(sA + i * kA), b0 = smem_addr(sB + i * 2 * kBp);
#pragma unroll
            for (uint32_t ks = 0; ks < kTcKBlock / 8; ++ks) {
                // A part: [k chunk 8][row group 16][8 x 16 B]: LBO 2048, SBO 128
                const uint64_t ahi = umma_desc(a0 + ks * 2 * 2048, 2048, 128);
                const uint64_t alo = umma_desc(a0 + kA / 2 + ks * 2 * 2048, 2048, 128);
                // B part: [k chunk 8][n group N/8][8 x 16 B]: LBO N*16, SBO 128
                const uint64_t bhi = umma_desc(b0 + ks * 2 * N * 16, N * 16, 128);
                const uint64_t blo = umma_desc(b0 + kBp + ks * 2 * N * 16, N * 16, 128);
                mma_tf32(tmem, ahi, bhi, idesc, (i | ks) != 0);
                mma_tf32(tmem, ahi, blo, idesc, 1u);
                mma_tf32(tmem, alo, bhi, idesc, 1u);
            }
        }
        mma_commit(bars + 1);
    }
    __syncwarp();
    bar_wait(bars + 1, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    CT_MARK(7);
    // epilogue: TMEM lane = centroid row (warp w owns lanes 32w..32w+31);
    // 32 columns per TMEM load
    const uint32_t c = tile * kTcRows + warp * 32 + lane;
    float* out = partial + size_t(blockIdx.z) * nq * nlist + size_t(q0) * nlist + c;
    const uint32_t trow = tmem + ((warp * 32) << 16);
    uint32_t j0 = 0;
    for (; j0 + 32 <= N; j0 += 32) {
        float v[32];
        tmem_ld32(trow + j0, v);
#pragma unroll
        for (uint32_t j = 0; j < 32; ++j)
            if (j0 + j < nvalid) out[size_t(j0 + j) * nlist] = v[j];
    }
    for (; j0 < N; j0 += 8) {
        float v[8];
        tmem_ld8(trow + j0, v);
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
            if (j0 + j < nvalid) out[size_t(j0 + j) * nlist] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
    CT_END(0);
}

// ------------------------------------------------------------------ K1b
constexpr uint32_t kWinThreads = 512;      // K1b block size when nq is large
constexpr uint32_t kWinThreadsMax = 1024;  // and its largest (SMEM reduction scratch is sized for it)
constexpr uint32_t kWinCap = 1024;   // window slots (ids + exact distances in SMEM)
constexpr uint32_t kStageRowsMax = 64;  // centroid rows staged per rescoring batch (fewer for large d)

__device__ __forceinline__ uint32_t fkey(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// nprobe-th smallest of the CTA's keys (rank is 1-based; keys in registers,
// VPT per thread, invalid slots hold 0xffffffff and are masked by `n`).
template <uint32_t VPT, uint32_t NT, class K>
__device__ K block_select_kth(const K (&key)[VPT], uint32_t n, uint32_t rank, uint32_t* hist, uint32_t* misc) {
    const uint32_t tid = threadIdx.x;
    K* sel = reinterpret_cast<K*>(misc + 2);  // selected prefix (misc[2..3])
    __syncthreads();
    if (tid == 0) {
        *sel = 0;
        misc[1] = rank;
    }
    K mask = 0;
    for (int shift = int(sizeof(K)) * 8 - 8; shift >= 0; shift -= 8) {
        for (uint32_t i = tid; i < 256; i += NT) hist[i] = 0;
        __syncthreads();
        const K prefix = *sel;
#pragma unroll
        for (uint32_t i = 0; i < VPT; ++i) {
            const bool act = (key[i] & mask) == prefix && i * NT + tid < n;
            const uint32_t bucket = uint32_t(key[i] >> shift) & 255u;
            const unsigned am = __ballot_sync(0xffffffffu, act);
            if (act) {
                const unsigned peers = __match_any_sync(am, bucket);
                if ((tid & 31) == uint32_t(__ffs(peers) - 1)) atomicAdd(&hist[bucket], __popc(peers));
            }
        }
        __syncthreads();
        if (tid < 32) {
            uint32_t v[8], local = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                v[i] = hist[tid * 8 + i];
                local += v[i];
            }
            uint32_t incl = local;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= uint32_t(o)) incl += t;
            }
            const uint32_t r = misc[1];
            const uint32_t excl = incl - local;
            if (excl < r && r <= incl) {
                uint32_t cacc = excl;
                int b = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (cacc + v[i] >= r) {
                        b = i;
                        break;
                    }
                    cacc += v[i];
                }
                misc[1] = r - cacc;
                *sel = prefix | (K(tid * 8 + b) << shift);
            }
        }
        __syncthreads();
        mask |= K(0xff) << shift;
    }
    return *sel;
}

// Appends every list c < n with pred(c) to win[] (order arbitrary); returns
// the count (may exceed kWinCap: only the first kWinCap are stored).
template <uint32_t NT, class Pred>
__device__ uint32_t block_collect(uint32_t n, Pred pred, uint32_t* win, uint32_t* counter) {
    const uint32_t tid = threadIdx.x;
    __syncthreads();
    if (tid == 0) *counter = 0;
    __syncthreads();
    const uint32_t span = (n + NT - 1) / NT * NT;
    for (uint32_t c = tid; c < span; c += NT) {
        const bool in = c < n && pred(c);
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        uint32_t base = 0;
        if ((tid & 31) == 0 && bal) base = atomicAdd(counter, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (in) {
            const uint32_t pos = base + __popc(bal & ((1u << (tid & 31)) - 1));
            if (pos < kWinCap) win[pos] = c;
        }
    }
    __syncthreads();
    return *counter;
}

// Exact fallback of K1b (window larger than kWinCap): the exact distance of
// every list into the query's scratch row, then selection on the unique
// (distance, list id) keys. Kept out of line: it never runs on well-posed
// inputs and would otherwise bloat the hot kernel's instruction footprint.
template <uint32_t VPT, uint32_t NT>
__device__ __noinline__ uint32_t exact_fallback(float* upq, const float* __restrict__ centroids, const float* sq,
                                                uint32_t nlist, uint32_t d, uint32_t nprobe, uint32_t* hist,
                                                uint32_t* misc, uint32_t* win, float* wd) {
    const uint32_t tid = threadIdx.x;
    uint32_t W;
        // fallback: exact distance of every list into this query's scratch row
    __syncthreads();
    for (uint32_t c = tid; c < nlist; c += NT) {
        const float* row = centroids + size_t(c) * d;
        float acc = 0.0f;
#pragma unroll 8
        for (uint32_t j = 0; j < d; ++j) {
            const float diff = __fsub_rn(sq[j], __ldg(row + j));
            acc = __fadd_rn(acc, __fmul_rn(diff, diff));
        }
        upq[c] = acc;
    }
    __syncthreads();
    // (distance, list id) composite keys are unique: the nprobe-th one
    // bounds a set of exactly nprobe lists
    uint64_t key64[VPT];
#pragma unroll
    for (uint32_t i = 0; i < VPT; ++i) {
        const uint32_t c = i * NT + tid;
        key64[i] = c < nlist ? (uint64_t(fkey(upq[c])) << 32 | c) : ~0ull;
    }
    const uint64_t tkey = block_select_kth<VPT, NT>(key64, nlist, nprobe, hist, misc);
    W = block_collect<NT>(nlist, [&](uint32_t c) { return (uint64_t(fkey(upq[c])) << 32 | c) <= tkey; }, win,
                      misc + 4);
    for (uint32_t i = tid; i < W; i += NT) wd[i] = upq[win[i]];
        return W;
}

// K1b. One CTA per query. Keys of A + E stay in registers (nlist <= 16384);
// U = the nprobe-th smallest by a 4-pass radix select; the window is rescored
// exactly and ranked. If the window exceeds kWinCap (not seen in practice:
// windows are nprobe + a few) the CTA falls back to the
// exact distance of every list and selects on the unique (distance, id) keys.
template <uint32_t VPT, uint32_t NT>  // lists per thread, threads: nlist <= VPT * NT
__global__ void __launch_bounds__(NT) select_window_kernel(
    float* __restrict__ partial, uint32_t nslices, const float* __restrict__ cent_norm, float bound_c,
    const float* __restrict__ centroids, const float* __restrict__ queries, uint32_t nq, uint32_t nlist, uint32_t d,
    uint32_t nprobe, uint32_t* __restrict__ probe, float* __restrict__ probe_dist,
    unsigned long long* __restrict__ win_stat, uint32_t kStageRows) {
    CT_BEGIN;
    // K2's CTAs (tables, planner) may take the SMs K1b leaves idle now: they
    // run their index-only prologue there and wait for this grid in
    // griddepcontrol.wait
    pdl_trigger();
    extern __shared__ __align__(1024) unsigned char sm[];
    uint32_t* hist = reinterpret_cast<uint32_t*>(sm);          // [256]
    uint32_t* misc = hist + 256;                               // [8]: [1] rank, [2..3] selected key, [4] count, [5..7] two-level U
    uint32_t* win = misc + 8;                                  // [kWinCap] list ids
    float* wd = reinterpret_cast<float*>(win + kWinCap);       // [kWinCap] exact distances
    float* sq = wd + kWinCap;                                  // [d] the query
    float* rows = sq + ((d + 3) & ~3u);                        // [2][kStageRows][d + 1] (kStageRows: launch arg)
    float* red = rows + 2 * kStageRows * (d + 1);              // [NT / 32] reduction scratch

    const uint32_t q = blockIdx.x, tid = threadIdx.x;
    // ||c||^2 is index data: load it before waiting on the previous kernel
    float cnv[VPT];
#pragma unroll
    for (uint32_t i = 0; i < VPT; ++i) {
        const uint32_t c = i * NT + tid;
        cnv[i] = c < nlist ? __ldg(cent_norm + c) : 0.0f;
    }
    // ||q||^2 (any order: it only enters the approximate A and the bound E).
    // The queries were written before K1 started, so they are read before
    // waiting on K1.
    float part = 0.0f;
    for (uint32_t j = tid; j < d; j += NT) {
        const float x = queries[size_t(q) * d + j];
        sq[j] = x;
        part = __fadd_rn(part, __fmul_rn(x, x));  // no FFMA anywhere in this kernel (SASS guard)
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((tid & 31) == 0) red[tid >> 5] = part;
    pdl_wait();
    CT_WAITED(1);
    // q.c: sum of K1's slices in slice order; up to ZB slices' loads are
    // issued together before the first add
    float dot[VPT];
#pragma unroll
    for (uint32_t i = 0; i < VPT; ++i) dot[i] = 0.0f;
    constexpr uint32_t ZB = VPT <= 8 ? 4 : 1;  // slices in flight (register budget)
    for (uint32_t z0 = 0; z0 < nslices; z0 += ZB) {
        float pv[ZB][VPT];
#pragma unroll
        for (uint32_t zz = 0; zz < ZB; ++zz) {
            const float* pz = partial + (size_t(z0 + zz) * nq + q) * nlist;
#pragma unroll
            for (uint32_t i = 0; i < VPT; ++i) {
                const uint32_t c = i * NT + tid;
                pv[zz][i] = (z0 + zz < nslices && c < nlist) ? pz[c] : 0.0f;
            }
        }
#pragma unroll
        for (uint32_t zz = 0; zz < ZB; ++zz)
            if (z0 + zz < nslices) {
#pragma unroll
                for (uint32_t i = 0; i < VPT; ++i) dot[i] += pv[zz][i];
            }
    }
    __syncthreads();
    float qn = 0.0f;
    for (uint32_t w = 0; w < NT / 32; ++w) qn += red[w];
    // A = ||q||^2 + ||c||^2 - 2 q.c; keys of A + E, and A - E
    uint32_t key[VPT];
    float lov[VPT];
#pragma unroll
    for (uint32_t i = 0; i < VPT; ++i) {
        const uint32_t c = i * NT + tid;
        key[i] = 0xffffffffu;
        lov[i] = 0.0f;
        if (c < nlist) {
            const float nrm = __fadd_rn(qn, cnv[i]);
            const float a = __fsub_rn(nrm, __fmul_rn(2.0f, dot[i]));
            const float e = __fmul_rn(bound_c, nrm);
            key[i] = fkey(__fadd_rn(a, e));
            lov[i] = __fsub_rn(a, e);
        }
    }
    CT_MARK(8);
    float* upq = partial + size_t(q) * nlist;  // slice-0 row: scratch for the exact fallback
    // U = the nprobe-th smallest key. Two levels when every thread holds
    // several keys: the nprobe-th smallest of the 512 per-thread minima is an
    // upper bound U' >= U (a subset's order statistic), so the keys <= U'
    // (about nprobe of them) contain the nprobe smallest; U is ranked among
    // those by counting. Falls back to the 4-pass radix select over all keys
    // when that candidate set is large.
    uint32_t ukey;
    if (VPT > 1) {
        uint32_t kmin[1] = {key[0]};
#pragma unroll
        for (uint32_t i = 1; i < VPT; ++i) kmin[0] = min(kmin[0], key[i]);
        uint32_t ub;
        if (nprobe <= 32) {
            // G >= nprobe groups of s lanes (s a power of two <= 32): the
            // nprobe-th smallest group minimum is itself >= U (an order
            // statistic of a subset), found by one warp ranking <= 32 values
            uint32_t sz = 32;
            while (sz > 1 && NT / (sz / 2) <= 32 && NT / sz < nprobe) sz >>= 1;
            // (NT / sz groups; sz = 32 gives 16 groups)
            const uint32_t G = NT / sz;
            uint32_t gm = kmin[0];
            for (uint32_t o = 1; o < sz; o <<= 1) gm = min(gm, __shfl_xor_sync(0xffffffffu, gm, o));
            if ((tid & (sz - 1)) == 0) hist[tid / sz] = gm;  // hist[] is free until the radix fallback
            __syncthreads();
            if (tid < 32) {
                const uint32_t lane = tid;
                const uint32_t v = lane < G ? hist[lane] : 0xffffffffu;
                uint32_t less = 0, eq = 0;
                for (uint32_t j = 0; j < 32; ++j) {
                    const uint32_t x = __shfl_sync(0xffffffffu, v, j);
                    less += x < v;
                    eq += x == v;
                }
                if (lane < G && less < nprobe && nprobe <= less + eq) misc[7] = v;
            }
            __syncthreads();
            ub = misc[7];
        } else {
            ub = block_select_kth<1, NT>(kmin, NT, nprobe, hist, misc);
        }
        uint32_t* cand = reinterpret_cast<uint32_t*>(wd);  // scratch until the window is rescored
        if (tid == 0) misc[5] = 0;
        __syncthreads();
#pragma unroll
        for (uint32_t i = 0; i < VPT; ++i) {
            const bool in = key[i] <= ub;
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            uint32_t base = 0;
            if ((tid & 31) == 0 && bal) base = atomicAdd(misc + 5, __popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (in) {
                const uint32_t pos = base + __popc(bal & ((1u << (tid & 31)) - 1));
                if (pos < kWinCap) cand[pos] = key[i];
            }
        }
        __syncthreads();
        const uint32_t nc = misc[5];
        if (nc <= kWinCap) {
            for (uint32_t i = tid; i < nc; i += NT) {
                const uint32_t ki = cand[i];
                uint32_t less = 0, eq = 0;
                for (uint32_t j = 0; j < nc; ++j) {
                    const uint32_t kj = cand[j];
                    less += kj < ki;
                    eq += kj == ki;
                }
                if (less < nprobe && nprobe <= less + eq) misc[6] = ki;
            }
            __syncthreads();
            ukey = misc[6];
        } else {
            ukey = block_select_kth<VPT, NT>(key, nlist, nprobe, hist, misc);
        }
    } else {
        ukey = block_select_kth<VPT, NT>(key, nlist, nprobe, hist, misc);
    }
    CT_MARK(9);
    // window: lists whose lower bound A - E does not exceed U
    // lov[] is in registers: collect through a per-thread test (c = i*512 + tid)
    uint32_t W;
    {
        __syncthreads();
        if (tid == 0) misc[4] = 0;
        __syncthreads();
#pragma unroll
        for (uint32_t i = 0; i < VPT; ++i) {
            const uint32_t c = i * NT + tid;
            const bool in = c < nlist && fkey(lov[i]) <= ukey;
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            uint32_t base = 0;
            if ((tid & 31) == 0 && bal) base = atomicAdd(misc + 4, __popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (in) {
                const uint32_t pos = base + __popc(bal & ((1u << (tid & 31)) - 1));
                if (pos < kWinCap) win[pos] = c;
            }
        }
        __syncthreads();
        W = misc[4];
        if (win_stat && tid == 0) atomicAdd(win_stat, (unsigned long long)W);
    }
    CT_MARK(10);
    const uint32_t rs = d + 1;
    if (W <= kWinCap) {
        // exact rescoring (common.hpp:73-80 via annindex.hpp:279): rows staged
        // in SMEM (stride d + 1: conflict-free) by cp.async; one thread folds
        // one list. A window that fits both staging buffers is staged and
        // folded as ONE batch (one fold chain instead of two in sequence);
        // larger ones go in batches of kStageRows, batch b+1 loading while
        // batch b is folded
        const uint32_t SB = W <= 2 * kStageRows ? 2 * kStageRows : kStageRows;
        auto stage_batch = [&](uint32_t b0, uint32_t buf) {
            const uint32_t nb = min(SB, W - b0);
            float* dst = rows + buf * kStageRows * rs;
            // warp w stages rows w, w + NT / 32, ...; lanes stride the row (no division)
            for (uint32_t r = tid >> 5; r < nb; r += NT / 32) {
                const float* src = centroids + size_t(win[b0 + r]) * d;
                const uint32_t drow = smem_addr(dst + r * rs);
                for (uint32_t j = tid & 31u; j < d; j += 32)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(drow + 4 * j), "l"(src + j)
                                 : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        if (W) stage_batch(0, 0);
        for (uint32_t b0 = 0, buf = 0; b0 < W; b0 += SB, buf ^= 1u) {
            const uint32_t nb = min(SB, W - b0);
            if (b0 + SB < W) {  // (SB = kStageRows here: two buffers in turn)
                stage_batch(b0 + SB, buf ^ 1u);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncthreads();
            if (tid < nb) {
                const float* row = rows + (buf * kStageRows + tid) * rs;
                float acc = 0.0f;
#pragma unroll 16
                for (uint32_t j = 0; j < d; ++j) {
                    const float diff = __fsub_rn(sq[j], row[j]);
                    acc = __fadd_rn(acc, __fmul_rn(diff, diff));
                }
                wd[b0 + tid] = acc;
            }
            __syncthreads();  // batch buffer free for the prefetch two batches on
        }
    } else {
        W = exact_fallback<VPT, NT>(upq, centroids, sq, nlist, d, nprobe, hist, misc, win, wd);
    }
    __syncthreads();
    CT_MARK(11);
    // rank by (distance, list id) (annindex.hpp:281 std::sort of pairs): one
    // warp per window list, its lanes counting the lists ordered before it
    {
        const uint32_t lane = tid & 31u;
        for (uint32_t i = tid >> 5; i < W; i += NT / 32) {
            const float di = wd[i];
            const uint32_t ci = win[i];
            uint32_t r = 0;
            for (uint32_t j = lane; j < W; j += 32) {
                const float dj = wd[j];
                r += (dj < di) || (dj == di && win[j] < ci);
            }
            r = __reduce_add_sync(0xffffffffu, r);
            if (lane == 0 && r < nprobe) {
                probe[size_t(q) * nprobe + r] = ci;
                probe_dist[size_t(q) * nprobe + r] = di;
            }
        }
    }
    CT_END(1);
}

}  // namespace

#ifdef PRAG_CHAIN_TRACE
CT_BIND_FN(ct_bind_coarse)
#endif

// rows per rescoring batch: up to kStageRowsMax while the double-buffered
// staging fits the 227 KiB opt-in (more rows fold in parallel for large nprobe)
static uint32_t window_stage_rows(uint32_t d) {
    const size_t fixed = (256 + 8 + 2 * kWinCap) * 4 + ((d + 3) & ~3u) * 4 + (kWinThreadsMax / 32) * 4;
    const size_t per_row = 2 * size_t(d + 1) * 4;
    const size_t fit = fixed < 227 * 1024 ? (227 * 1024 - fixed) / per_row : 0;
    return uint32_t(std::min<size_t>(kStageRowsMax, fit));
}

size_t tc_window_smem(uint32_t d) {
    const uint32_t rows = std::max<uint32_t>(window_stage_rows(d), 8);
    return (256 + 8 + 2 * kWinCap) * 4 + ((d + 3) & ~3u) * 4 + 2 * size_t(rows) * (d + 1) * 4 +
           (kWinThreadsMax / 32) * 4;
}

bool tc_coarse_supported(uint32_t nlist, uint32_t d) {
    return nlist % kTcRows == 0 && nlist <= 32 * kWinThreads && d % kTcKBlock == 0 &&
           d <= kTcMaxSlices * kTcSliceBlocks * kTcKBlock &&
           tc_window_smem(d) <= 227 * 1024;
}

float tc_bound_c(uint32_t d) { return float((8.0 * d + 256.0) * 0x1p-24); }

// K1's A operand, host-side: the fp32 centroids per 128-row tile and
// 32-element K block in [k chunk 8][row group 16][8 rows][4] order (the
// no-swizzle K-major core-matrix layout); K1 splits each staged block into
// its hi and lo parts in SMEM.
void build_tc_centroids(const float* cent, uint32_t nlist, uint32_t d, std::vector<float>& out,
                        std::vector<float>& norms) {
    const uint32_t tiles = nlist / kTcRows, nkb = d / kTcKBlock;
    out.assign(size_t(nlist) * d, 0.0f);
    norms.resize(nlist);
    for (uint32_t c = 0; c < nlist; ++c) {
        double s = 0.0;
        for (uint32_t j = 0; j < d; ++j) s += double(cent[size_t(c) * d + j]) * cent[size_t(c) * d + j];
        norms[c] = float(s);
    }
    for (uint32_t t = 0; t < tiles; ++t)
        for (uint32_t kb = 0; kb < nkb; ++kb) {
            float* blk = out.data() + (size_t(t) * nkb + kb) * (kTcRows * kTcKBlock);
            for (uint32_t r = 0; r < kTcRows; ++r)
                for (uint32_t k = 0; k < kTcKBlock; ++k) {
                    const size_t off = size_t(k >> 2) * (kTcRows * 4) + (r >> 3) * 32 + (r & 7) * 4 + (k & 3);
                    blk[off] = cent[size_t(t * kTcRows + r) * d + kb * kTcKBlock + k];
                }
        }
}

uint32_t tc_slices(uint32_t d) { return (d / kTcKBlock + kTcSliceBlocks - 1) / kTcSliceBlocks; }

int launch_coarse_tc(const DeviceIndex& ix, const float* queries, uint32_t nq, float* partial, cudaStream_t s) {
    const uint32_t n_tile = std::min<uint32_t>(kTcMaxN, (nq + 7) / 8 * 8);
    const size_t kA = 2 * kTcRows * kTcKBlock * 4, kBp = size_t(n_tile) * kTcKBlock * 4;
    const size_t smem = kTcSliceBlocks * kA + kTcSliceBlocks * 2 * kBp + 2 * 8 + 16;
    PG_CUDA(ensure_smem(reinterpret_cast<const void*>(coarse_tc_kernel), int(smem)));
    dim3 grid(ix.nlist / kTcRows, (nq + n_tile - 1) / n_tile, tc_slices(ix.d));
    cudaError_t e = launch_pdl(coarse_tc_kernel, grid, dim3(128), smem, s, ix.cent_tc, queries, nq, ix.nlist, ix.d,
                               n_tile, partial);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("CUDA launch failed (coarse_tc): ") + cudaGetErrorString(e));
        return PRAG_GPU_CUDA;
    }
    return PRAG_GPU_OK;
}

// K1b block size for this shape (see launch_select_window).
static uint32_t k1b_threads(uint32_t nlist, uint32_t nq) {
    (void)nq;
    return nlist > 2 * kWinThreads ? kWinThreadsMax : kWinThreads;
}

int launch_select_window(const DeviceIndex& ix, float* partial, const float* queries, uint32_t nq, uint32_t nprobe,
                         uint32_t* probe, float* probe_dist, unsigned long long* win_stat, cudaStream_t s) {
    const size_t smem = tc_window_smem(ix.d);
#define PG_WIN(V, T)                                                                                           \
    do {                                                                                                       \
        PG_CUDA(ensure_smem(reinterpret_cast<const void*>(select_window_kernel<V, T>), int(smem)));             \
        PG_CUDA(launch_pdl(select_window_kernel<V, T>, dim3(nq), dim3(T), smem, s, partial, tc_slices(ix.d),     \
                           ix.cent_norm, tc_bound_c(ix.d), ix.centroids, queries, nq, ix.nlist, ix.d, nprobe, probe, \
                           probe_dist, win_stat, std::max<uint32_t>(window_stage_rows(ix.d), 8)));              \
    } while (0)
    // Block size: the per-query CTA's phases (slice sums, U, window, ranking)
    // are latency chains over VPT keys per thread, so fewer keys per thread
    // shortens them. PRAG_GPU_K1B_THREADS (512 / 1024) overrides (A/B knob).
    const char* te = getenv("PRAG_GPU_K1B_THREADS");
    const uint32_t nt = te ? (atoi(te) >= 1024 ? 1024u : 512u) : k1b_threads(ix.nlist, nq);
    const uint32_t vpt = (ix.nlist + nt - 1) / nt;
    if (nt == 1024) {
        if (vpt <= 2)
            PG_WIN(2, 1024);
        else if (vpt <= 4)
            PG_WIN(4, 1024);
        else if (vpt <= 8)
            PG_WIN(8, 1024);
        else
            PG_WIN(16, 1024);
    } else if (vpt <= 2)
        PG_WIN(2, 512);
    else if (vpt <= 4)
        PG_WIN(4, 512);
    else if (vpt <= 8)
        PG_WIN(8, 512);
    else if (vpt <= 16)
        PG_WIN(16, 512);
    else
        PG_WIN(32, 512);
#undef PG_WIN
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("CUDA launch failed (select_window): ") + cudaGetErrorString(e));
        return PRAG_GPU_CUDA;
    }
    return PRAG_GPU_OK;
}

}  // namespace pg
