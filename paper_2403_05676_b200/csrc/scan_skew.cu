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
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "internal.h"
#include "skew_common.cuh"

namespace pg {
namespace {

using namespace skew;
constexpr uint32_t kMaxItemTiles = 512;  // tiles per scan work item (16384 entries) at most
constexpr uint32_t kMinItemTiles = 32;   // and at least (small batches: more, smaller items)

// ----------------------------------------------------------- LUT images
// {(r0 - w)^2, (r1 - w)^2}: one FADD2 then one FMUL2, each lane a single
// rounding (= __fsub_rn then __fmul_rn). The fold's adds stay scalar FADD:
// ptxas contracts a packed mul followed by a packed add into FFMA2, but never
// a packed mul into a scalar add.
__device__ __forceinline__ void subsq2_bcast(float r0, float r1, float w, float& s0, float& s1) {
    unsigned long long out;
    asm("{.reg .b64 A, B, D;\n"
        " mov.b64 A, {%1, %2};\n"
        " mov.b64 B, {%3, %3};\n"
        " sub.rn.f32x2 D, A, B;\n"
        " mul.rn.f32x2 %0, D, D;}"
        : "=l"(out)
        : "f"(r0), "f"(r1), "f"(w));
    s0 = __uint_as_float(uint32_t(out));
    s1 = __uint_as_float(uint32_t(out >> 32));
}

// SMEM image of one (query, list) ADC table, as K3 gathers it: R = m/32
// images of [256 codes][64 columns] fp32 (64 KiB each). Lane t at fold step
// s reads column s - t + 32 of image s/32, so with
//   image 0:      column c holds T[(c - 32) mod m]
//   image r >= 1: column c holds T[c + 32 (r - 1)]
// every step's 32 lanes hit 32 distinct banks whatever the code bytes are.
// The LUT kernel writes the compact table T[sq][256] (coalesced); K3's
// expander warps build the image from it in SMEM.
template <int M>
constexpr uint32_t image_floats() {
    return uint32_t(M / 32) * 256u * 64u;
}

// Work items for the fast path: per (q, p) pair, ceil(len/32) tiles cut into
// items of <= it_tiles tiles, emitted largest-first (a counting sort on the
// item's tile count) so the big lists set each query's threshold early, the
// small ones fill the tail, and the persistent CTAs, which pull items a few
// ahead of scanning them, finish together. q_item_off[q] = prefix of per-query item counts (candidate-pool
// offsets). Also resets the per-query threshold and pool counters, and
// writes scanned_vectors (annindex.hpp:305: the sum of probed list sizes).
struct PlanArgs {
    uint32_t it_tiles;
    uint32_t split_items;  // full items cut into kSplit smaller ones (scheduled last): the queue's tail
    uint64_t* scanned;
    uint4* items;
    uint32_t* num_items;
    uint32_t* cursor;
    uint32_t* q_item_off;
    uint32_t* gthr;
    uint32_t* pair_off;  // [nq * nprobe] pool item index of each pair's first item
    uint64_t item_cap;
};

// The scan's work queue is consumed largest item first, so the kernel's tail
// is the last items: with ~4 items per CTA of up to kMaxItemTiles each (config
// C/D at batch 1) a CTA can finish a whole item after the others. The planner
// therefore cuts `split_items` of the full items into kSplit pieces that land
// in a smaller size bucket, i.e. at the end of the queue ("guided" tail).
constexpr uint32_t kSplit = 4;

// Fire-and-forget 64-bit add to global memory (a plain atomicAdd on a generic
// pointer compiles to a blocking generic atomic with a shared-memory CAS
// fallback).
__device__ __forceinline__ void red_add_u64(uint64_t* p, uint64_t v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
}

// pos[b] = sum of cnt[b'] over b' > b (b < nb): bucket start positions with
// the largest bucket first. Called by the whole block; ends synchronised.
__device__ __forceinline__ void desc_positions(const uint32_t* cnt, uint32_t* pos, uint32_t nb, uint32_t* ws) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, w = tid >> 5, nw = blockDim.x >> 5;
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;  // reversed buckets [tid*per, +per) per thread
    __syncthreads();  // counts complete
    uint32_t local = 0;
    for (uint32_t j = 0; j < per; ++j) {
        const uint32_t r = tid * per + j;
        if (r < nb) local += cnt[nb - 1 - r];
    }
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += t;
    }
    if (lane == 31) ws[w] = incl;
    __syncthreads();
    if (w == 0) {
        const uint32_t x = lane < nw ? ws[lane] : 0u;
        uint32_t xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= uint32_t(o)) xi += t;
        }
        if (lane < nw) ws[lane] = xi - x;
    }
    __syncthreads();
    uint32_t run = ws[w] + incl - local;
    for (uint32_t j = 0; j < per; ++j) {
        const uint32_t r = tid * per + j;
        if (r < nb) {
            pos[nb - 1 - r] = run;
            run += cnt[nb - 1 - r];
        }
    }
    __syncthreads();
}

// plan_items for up to R pairs per thread (P <= R * blockDim.x): thread t
// owns pairs [t*R, t*R + R), so every probe[] / list_len[] load is issued up
// front (two dependent rounds in all), the pair-order prefix is one serial
// sum per thread plus one block scan, and the scatter reuses the registers.
// Same outputs as plan_items.
// dry: the same instruction stream with no memory reads or global writes (one
// tile per pair). The planner CTA runs it before waiting on K1b: K2's CTAs
// launch early (K1b triggers at its start), and the planner is one CTA
// running this code once, so otherwise nearly every instruction line is an
// instruction-cache miss (measured: most of its ~17 us was no_instruction
// stalls at nq 64, nprobe 16).
template <int R>
__device__ __noinline__ void plan_items_regs(const uint32_t* __restrict__ probe, const uint32_t* __restrict__ list_len,
                                             uint32_t nq, uint32_t nprobe, const PlanArgs pa, bool dry) {
    CT_BEGIN;
    const uint32_t it_tiles = pa.it_tiles;
    __shared__ uint32_t wsum[33], bws[33];
    __shared__ uint32_t bucket_cnt[kMaxItemTiles + 1], bucket_pos[kMaxItemTiles + 1];
    const uint32_t P = nq * nprobe, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t nb = it_tiles + 1;  // one bucket per item size (tiles)
    for (uint32_t b = tid; b < nb; b += blockDim.x) bucket_cnt[b] = 0;
    if (!dry)
        for (uint32_t q = tid; q < nq; q += blockDim.x) {
            pa.scanned[q] = 0;
            pa.gthr[q] = 0xffffffffu;
        }
    uint32_t len[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = tid * R + r;
        len[r] = i < P && !dry ? probe[i] : 0u;  // list id for now
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = tid * R + r;
        len[r] = i < P ? (dry ? kTileEntries : list_len[len[r]]) : 0u;
    }
    CT_MARK(12);
    // full items of this thread's pairs, and their exclusive prefix over the
    // block (pair order): full item number g < split is cut into kSplit pieces
    uint32_t fmine = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t tiles = (len[r] + kTileEntries - 1) / kTileEntries;
        const uint32_t nit = (tiles + it_tiles - 1) / it_tiles;
        fmine += nit ? nit - 1 : 0u;
    }
    const uint32_t split = it_tiles >= kSplit * kMinItemTiles ? pa.split_items : 0u;
    uint32_t fincl = fmine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, fincl, o);
        if (lane >= uint32_t(o)) fincl += t;
    }
    if (lane == 31) wsum[w] = fincl;
    __syncthreads();  // scanned[] zeroed, bucket_cnt ready, full-item warp sums
    if (w == 0) {
        const uint32_t nw = blockDim.x >> 5;
        const uint32_t x = lane < nw ? wsum[lane] : 0u;
        uint32_t xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= uint32_t(o)) xi += t;
        }
        if (lane < nw) wsum[lane] = xi - x;
    }
    __syncthreads();
    const uint32_t fexcl0 = wsum[w] + fincl - fmine;
    __syncthreads();  // wsum is reused below
    CT_MARK(13);
    const uint32_t sub_tiles = it_tiles / kSplit;
    uint32_t mine = 0;
    {
        uint32_t fexcl = fexcl0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t i = tid * R + r;
            if (len[r] && !dry) red_add_u64(pa.scanned + i / nprobe, len[r]);
            const uint32_t tiles = (len[r] + kTileEntries - 1) / kTileEntries;
            const uint32_t nit = (tiles + it_tiles - 1) / it_tiles;
            if (nit) {  // nit - 1 full items (the first `split - fexcl` of them cut), then the remainder
                const uint32_t full = nit - 1;
                const uint32_t cut = fexcl < split ? min(full, split - fexcl) : 0u;
                if (full > cut) atomicAdd(&bucket_cnt[it_tiles], full - cut);
                if (cut) atomicAdd(&bucket_cnt[sub_tiles], cut * kSplit);
                atomicAdd(&bucket_cnt[tiles - full * it_tiles], 1u);
                mine += nit + cut * (kSplit - 1);
                fexcl += full;
            }
        }
    }
    // exclusive block prefix of `mine` (pair order = thread order)
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += t;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        const uint32_t nw = blockDim.x >> 5;
        const uint32_t x = lane < nw ? wsum[lane] : 0u;
        uint32_t xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= uint32_t(o)) xi += t;
        }
        if (lane < nw) wsum[lane] = xi - x;
        if (lane == nw - 1) wsum[32] = xi;
    }
    desc_positions(bucket_cnt, bucket_pos, nb, bws);
    __syncthreads();
    CT_MARK(14);
    uint32_t excl = wsum[w] + incl - mine;
    uint32_t fexcl = fexcl0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = tid * R + r;
        if (i >= P) break;
        if (!dry) {
            pa.pair_off[i] = excl;
            if (i % nprobe == 0) pa.q_item_off[i / nprobe] = excl;
        }
        const uint32_t tiles = (len[r] + kTileEntries - 1) / kTileEntries;
        const uint32_t nit = (tiles + it_tiles - 1) / it_tiles;
        uint32_t nout = 0;  // items this pair emits (pool slots excl .. excl + nout)
        if (nit) {
            const uint32_t full = nit - 1;
            const uint32_t cut = fexcl < split ? min(full, split - fexcl) : 0u;
            // the first `cut` full items in kSplit pieces (the queue's tail)
            const uint32_t c0 = cut ? atomicAdd(&bucket_pos[sub_tiles], cut * kSplit) : 0u;
            for (uint32_t j = 0; j < cut; ++j)
                for (uint32_t h = 0; h < kSplit; ++h) {
                    const uint32_t tb = j * it_tiles + h * sub_tiles, n = j * kSplit + h;
                    if (c0 + n < pa.item_cap && !dry) pa.items[c0 + n] = make_uint4(i, tb, tb + sub_tiles, excl + n);
                }
            nout = cut * kSplit;
            const uint32_t b0 = full > cut ? atomicAdd(&bucket_pos[it_tiles], full - cut) : 0u;
            for (uint32_t j = cut; j < full; ++j) {
                const uint32_t n = b0 + (j - cut);
                if (n < pa.item_cap && !dry) pa.items[n] = make_uint4(i, j * it_tiles, (j + 1) * it_tiles, excl + nout);
                ++nout;
            }
#ifdef PRAG_EXP_NOATOM
            const uint32_t slot = i;
#else
            const uint32_t slot = atomicAdd(&bucket_pos[tiles - full * it_tiles], 1u);
#endif
#ifndef PRAG_EXP_NOSTORE
            if (slot < pa.item_cap && !dry) pa.items[slot] = make_uint4(i, full * it_tiles, tiles, excl + nout);
#endif
            ++nout;
            fexcl += full;
        }
        excl += nout;
        if (r == 0) CT_MARK(16);
        if (r == 1) CT_MARK(17);
        if (r == 2) CT_MARK(18);
    }
    if (tid == 0 && !dry) {
        *pa.num_items = wsum[32];
        *pa.cursor = 0;
        pa.q_item_off[nq] = wsum[32];
    }
    CT_MARK(15);
}

// Runs on one CTA (any block size that is a multiple of 32, <= 1024): the
// extra CTA of the LUT kernel's grid, so planning overlaps the LUT work.
__device__ __noinline__ void plan_items(const uint32_t* __restrict__ probe, const uint32_t* __restrict__ list_len,
                                        uint32_t nq, uint32_t nprobe, const PlanArgs pa) {
    const uint32_t it_tiles = pa.it_tiles;
    uint64_t* __restrict__ scanned = pa.scanned;
    uint4* __restrict__ items = pa.items;
    uint32_t* __restrict__ num_items = pa.num_items;
    uint32_t* __restrict__ cursor = pa.cursor;
    uint32_t* __restrict__ q_item_off = pa.q_item_off;
    uint32_t* __restrict__ gthr = pa.gthr;
    uint32_t* __restrict__ pair_off = pa.pair_off;
    const uint64_t item_cap = pa.item_cap;
    __shared__ uint32_t tmp[33], bws[33];
    __shared__ uint32_t bucket_cnt[kMaxItemTiles + 1], bucket_pos[kMaxItemTiles + 1];
    const uint32_t P = nq * nprobe;
    const uint32_t nb = it_tiles + 1;  // one bucket per item size (tiles)
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) bucket_cnt[b] = 0;
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) scanned[q] = 0;
    __syncthreads();
    // pass 1: per-query item counts (prefix) and bucket histogram
    uint32_t carry = 0;
    for (uint32_t base = 0; base < P; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const bool valid = i < P;
        const uint32_t len = valid ? list_len[probe[i]] : 0;
        if (len) red_add_u64(scanned + i / nprobe, len);
        const uint32_t tiles = (len + kTileEntries - 1) / kTileEntries;
        const uint32_t nit = (tiles + it_tiles - 1) / it_tiles;
        for (uint32_t j = 0; j < nit; ++j) {
            const uint32_t t = min(tiles, (j + 1) * it_tiles) - j * it_tiles;
            atomicAdd(&bucket_cnt[t], 1u);
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
        if (valid) pair_off[i] = excl;
        if (valid && i % nprobe == 0) q_item_off[i / nprobe] = excl;
        carry += tmp[32];
        __syncthreads();
    }
    // bucket start positions, largest item first
    desc_positions(bucket_cnt, bucket_pos, nb, bws);
    // pass 2: scatter items
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        const uint32_t len = list_len[probe[i]];
        const uint32_t tiles = (len + kTileEntries - 1) / kTileEntries;
        const uint32_t nit = (tiles + it_tiles - 1) / it_tiles;
        for (uint32_t j = 0; j < nit; ++j) {
            const uint32_t te = min(tiles, (j + 1) * it_tiles);
            const uint32_t slot = atomicAdd(&bucket_pos[te - j * it_tiles], 1u);
            // .w: the item's slot in the candidate pool (pair order, so a query's
            // items are contiguous: [q_item_off[q], q_item_off[q + 1]))
            if (slot < item_cap) items[slot] = make_uint4(i, j * it_tiles, te, pair_off[i] + j);
        }
    }
    if (threadIdx.x == 0) {
        *num_items = carry;
        *cursor = 0;
        q_item_off[nq] = carry;
    }
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) gthr[q] = 0xffffffffu;
}


// The planner CTA of K2 (the grid's last block): work items of the scan.
__device__ __forceinline__ void planner_cta(const uint32_t* __restrict__ probe, const uint32_t* __restrict__ list_len,
                                            uint32_t nq, uint32_t nprobe, const PlanArgs& pa) {
    CT_BEGIN;
    const uint32_t P = nq * nprobe;
    const int R = P <= blockDim.x ? 1 : P <= 4 * blockDim.x ? 4 : P <= 8 * blockDim.x ? 8 : 0;
    for (int pass = 0; pass < 2; ++pass) {  // 0: instruction-cache warm-up (dry), 1: the plan
        const bool dry = pass == 0;
        if (!dry) {
            pdl_wait();  // probe[] comes from the previous kernel
            CT_WAITED(3);
        }
        if (R == 1)
            plan_items_regs<1>(probe, list_len, nq, nprobe, pa, dry);
        else if (R == 4)
            plan_items_regs<4>(probe, list_len, nq, nprobe, pa, dry);
        else if (R == 8)
            plan_items_regs<8>(probe, list_len, nq, nprobe, pa, dry);
        else if (!dry)
            plan_items(probe, list_len, nq, nprobe, pa);
    }
}

// K2: the ADC tables T[pair][sq][256] (annindex.hpp:292-297: squared_l2 of
// the residual r = q - c_list (annindex.hpp:287-289) against every codeword
// of subquantizer sq) as a persistent kernel: G table CTAs (two per SM of the
// search's SM budget, less one for the planner) + the planner CTA (block 0).
// Task t = (chunk of
// kTaskPairs pairs t / m, subquantizer t % m); CTA c takes tasks c, c + G, ...
// (equal cost: static). Thread = code: its codeword w[sq][code][0..sub) comes
// from the transposed codebook (coalesced); the task's residuals sit in SMEM as
// [j][pair], so one LDS.128 broadcasts four pairs. Software pipeline per task:
// the next task's codewords and residual inputs, and the list ids of the task
// after it, load while this task is folded, so no CTA waits on memory between
// tasks (the one-task-per-CTA form paid a launch-and-load prologue per CTA
// and a partial last wave: ~17.5 us at config B vs ~8 us of FP32 work).
constexpr uint32_t kTaskPairs = 16;
template <int M, int SUBC>  // SUBC: compile-time sub_dim (0 = runtime `sub`, <= 16)
__global__ void __launch_bounds__(256, 2) lut_tasks_kernel(const float* __restrict__ queries,
                                                           const float* __restrict__ centroids,
                                                           const float* __restrict__ codewordsT,
                                                           const uint32_t* __restrict__ probe,
                                                           const uint32_t* __restrict__ list_len, uint32_t nq,
                                                           uint32_t nprobe, uint32_t d, uint32_t sub,
                                                           float* __restrict__ luts, const PlanArgs pa) {
    CT_BEGIN;
    if (blockIdx.x == 0) {  // block 0: launched first, so it never waits for an SM
        planner_cta(probe, list_len, nq, nprobe, pa);
        CT_END(3);
        return;
    }
    constexpr uint32_t P = kTaskPairs;
    constexpr int JMAX = SUBC ? SUBC : 16;
    if (SUBC) sub = SUBC;
    __shared__ __align__(16) float resid[2][16 * P];  // [buffer][j][pair]
    const uint32_t npairs = nq * nprobe;
    const uint32_t nchunks = (npairs + P - 1) / P;
    const uint32_t ntasks = nchunks * M;
    const uint32_t G = gridDim.x - 1, code = threadIdx.x, tid = threadIdx.x;
    // residual-input role of this thread: pair pl of the task, dimension jj
    const bool rin = tid < P * sub;
    const uint32_t pl = rin ? tid / sub : 0u, jj = rin ? tid - pl * sub : 0u;
    uint32_t t = blockIdx.x - 1;
    if (t >= ntasks) {
        pdl_trigger();
        return;
    }
    // task t's codewords first (index data, before the dependency wait)
    float w[JMAX];
#pragma unroll
    for (int j = 0; j < JMAX; ++j)
        if (j < int(sub)) w[j] = __ldg(codewordsT + (size_t(t % M) * sub + j) * 256 + code);
    pdl_wait();  // probe[] comes from the previous kernel
    CT_WAITED(2);
    // list id of this thread's pair in task t and in task t + G
    auto list_of = [&](uint32_t task) -> uint32_t {
        const uint32_t pair = (task / M) * P + pl;
        return (rin && task < ntasks && pair < npairs) ? probe[pair] : 0xffffffffu;
    };
    auto resid_in = [&](uint32_t task, uint32_t list, float& qv, float& cv) {
        qv = cv = 0.0f;
        if (list != 0xffffffffu) {
            const uint32_t pair = (task / M) * P + pl, dim = (task % M) * sub + jj;
            qv = queries[size_t(pair / nprobe) * d + dim];
            cv = centroids[size_t(list) * d + dim];
        }
    };
    uint32_t lcur = list_of(t), lnext = list_of(t + G);
    float qv, cv;
    resid_in(t, lcur, qv, cv);
    uint32_t buf = 0;
    for (;;) {
        // residuals of task t (tables of empty lists are computed too: the
        // scan never reads them)
        if (rin) resid[buf][jj * P + pl] = lcur != 0xffffffffu ? __fsub_rn(qv, cv) : 0.0f;
        __syncthreads();
        // next task's inputs, loaded while this one is folded
        const uint32_t tn = t + G;
        float wn[JMAX];
        float qn = 0.0f, cn = 0.0f;
        uint32_t lnn = 0xffffffffu;
        if (tn < ntasks) {
#pragma unroll
            for (int j = 0; j < JMAX; ++j)
                if (j < int(sub)) wn[j] = __ldg(codewordsT + (size_t(tn % M) * sub + j) * 256 + code);
            resid_in(tn, lnext, qn, cn);
            lnn = list_of(tn + G);
        }
        const uint32_t p0 = (t / M) * P, sq = t % M;
        const uint32_t nlive = min(P, npairs - p0);
        const float* rr = resid[buf];
#pragma unroll 1
        for (uint32_t c = 0; c < P / 8; ++c) {
            if (c * 8 >= nlive) break;
            // FADD2 (r - w) and FMUL2 (square) two pairs at a time, scalar
            // FADD accumulation in j order: every step separately rounded, no
            // FMUL2 -> FADD2 pair for ptxas to contract into an FFMA2 (the
            // first term is the accumulator itself: 0 + x = x exactly)
            float acc[8];
#pragma unroll
            for (int j = 0; j < JMAX; ++j) {
                if (j < int(sub)) {
                    const float4 ra = *reinterpret_cast<const float4*>(rr + j * P + c * 8);
                    const float4 rb = *reinterpret_cast<const float4*>(rr + j * P + c * 8 + 4);
                    float sqv[8];  // fl(fl(r - w)^2)
                    subsq2_bcast(ra.x, ra.y, w[j], sqv[0], sqv[1]);
                    subsq2_bcast(ra.z, ra.w, w[j], sqv[2], sqv[3]);
                    subsq2_bcast(rb.x, rb.y, w[j], sqv[4], sqv[5]);
                    subsq2_bcast(rb.z, rb.w, w[j], sqv[6], sqv[7]);
#pragma unroll
                    for (int p = 0; p < 8; ++p) acc[p] = j == 0 ? sqv[p] : __fadd_rn(acc[p], sqv[p]);
                }
            }
            float* dst = luts + (size_t(p0 + c * 8) * M + sq) * 256 + code;
#pragma unroll
            for (int p = 0; p < 8; ++p)
                if (c * 8 + p < nlive) dst[size_t(p) * M * 256] = acc[p];
        }
        if (tn >= ntasks) break;
        t = tn;
#pragma unroll
        for (int j = 0; j < JMAX; ++j) w[j] = wn[j];
        qv = qn;
        cv = cn;
        lcur = lnext;
        lnext = lnn;
        buf ^= 1u;
    }
    pdl_trigger();
    CT_END(2);
}

// ------------------------------------------------------------------- scan
template <int M>
struct SkewCfg;
template <>
struct SkewCfg<32> {
    // consumer warps; + 1 producer + kExp expander warps, 1 CTA per SM
    // (12 + 3 measured best with the SMEM code ring: 13 + 2 138.6 us, 12 + 3
    // 132.1, 11 + 4 140.1 at config B)
    static constexpr int kWarps = 12;
    static constexpr int kExp = 3;
    static constexpr int kPrefetch = 2;  // tiles a warp keeps requested into L2 ahead of its loads (2-16 measured within 2%)
};
template <>
struct SkewCfg<64> {
    // 10 consumers + producer + 1 expander = 12 warps, 3 per SM
    // sub-partition: up to 168 registers a thread, so both code tiles in
    // flight (32 registers) and the 64 step-mask registers stay resident
    // (with 15 warps the 128-register cap made ptxas rematerialise the masks
    // inside the fold, ~35 extra instructions per 2 KiB tile)
    static constexpr int kWarps = 10;
    static constexpr int kExp = 1;
    static constexpr int kPrefetch = 2;
};

constexpr uint32_t kEndItem = 0xffffffffu;

#ifdef PRAG_K3_TRACE
// Debug build only (make EXTRA=-DPRAG_K3_TRACE): per-CTA globaltimer events of
// K3 -- [0] after pdl_wait, then per item consumed by warp 0: (start, end,
// tiles), finally the exit time. Read back with prag_gpu_debug_k3_trace.
constexpr uint32_t kTraceSlots = 256;
__device__ unsigned long long g_k3_trace[160 * kTraceSlots];
// per CTA, per item (< 32): [0] producer has the item's info, [1] producer
// issued its table copy, [2] expander 0 saw the table staged, [3] expander 0
// got the image buffer, [4] image ready, [5] last consumer warp done with it
__device__ unsigned long long g_k3_trace2[160 * 6 * 32];
#define K3T2(kind, idx, t)                                                                        \
    do {                                                                                          \
        if ((idx) < 32u) g_k3_trace2[(size_t(blockIdx.x) * 6 + (kind)) * 32 + (idx)] = (t);        \
    } while (0)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif
constexpr uint32_t kMinWarpTiles = 4;  // a warp re-reads one tail tile per range: keep ranges >= 4 tiles
constexpr uint32_t kHeadTiles = 4;     // first tiles of each warp range the producer requests into L2

struct ItemSlot {
    uint32_t pair, tb, te, len, q;
    uint32_t thr;            // the query's shared threshold when the producer fetched the item
    uint32_t pslot;          // the item's slot in the query's candidate pool (k entries each)
    uint64_t tile_byte_off;  // skew_off[list] * tile bytes
    uint64_t lbase;          // list_off[list]: padded entry slot of the list's entry 0
};

// SMEM plan of K3: two LUT images (item i+1's is built while item i is
// scanned), the staging buffer the producer bulk-copies compact tables into,
// then barriers, item slots and the merge stashes. Image 0 starts at a
// 64 KiB-aligned shared address and image 1 a fixed stride above it, so a
// gather address is PRMT(code byte -> bits 8..15, lane column -> bits 0..7,
// image page -> bits 16..31) plus a compile-time offset: one PRMT and one
// LDS [R + imm] per code byte. The staging buffer and the tail go into the
// alignment pad below image 0 when they fit there, else above the images.
//  * m = 32: image [256 codes][64 columns] fp32, column c = T[c mod 32] (the
//    wrap-around duplicated), lane t at step s reads column 32 + s - t.
//  * m = 64: image [256][64], column c = T[c] (no duplicate), lane t at step
//    s reads column (s - t) mod 64. The wrap (s < t: the tail of the previous
//    entry) is folded into the code byte: the ingest stores those bytes as
//    (code + 1) mod 256, so row code + 1 minus 4(t - s) bytes lands on column
//    64 + s - t of row `code`. Code 255 wraps to row 0 and reads just below
//    the image: a 128-byte guard holding row 255's upper half.
// Code tiles are not staged in SMEM at all: each lane loads the 16-byte
// chunks it folds straight into registers, one tile ahead, and lane 0 keeps
// the warp's next kPrefetch tiles requested into L2 (bulk prefetch).
template <int M>
struct SkewSmem {
    static constexpr int W = SkewCfg<M>::kWarps, NB = 2;
    static constexpr uint32_t kGuard = M == 64 ? 128u : 0u;
    static constexpr uint32_t kImg = 65536;
    static constexpr uint32_t kImgStride = kGuard + kImg;
    static constexpr uint32_t kStage = 32768;  // 32 subquantizers of T[sq][256] fp32
    // img_full[NB], stg_full
    static constexpr uint32_t nbars = NB + 1;
    // + cta_thr[NB] + merge counters[NB] + per-(buffer, warp) list stash {key[32], pos[32]}
    static constexpr uint32_t kTail = 8 * nbars + (NB + 1) * uint32_t(sizeof(ItemSlot)) + 4 * NB + 4 * NB +
                                      uint32_t(NB) * W * 64 * 4;
    static constexpr uint32_t kImgSpan = kImgStride + kImg;  // image 0 start .. image 1 end
    static constexpr uint32_t bytes = 232448;                 // 227 KiB: the opt-in maximum
    // worst case: a pad just too small for the staging buffer and the tail
    static constexpr uint32_t worst = (kGuard + kStage + kTail - 16) + kImgSpan + kStage + kTail;
    static constexpr int threads = (W + 1 + SkewCfg<M>::kExp) * 32;
};

template <int M>
constexpr size_t skew_smem_bytes() {
    return SkewSmem<M>::bytes;
}
static_assert(SkewSmem<32>::worst <= SkewSmem<32>::bytes && SkewSmem<64>::worst <= SkewSmem<64>::bytes,
              "K3 SMEM exceeds 227 KiB");

struct ScanCtx {
    uint32_t* cta_thr;  // this item's CTA-wide threshold (SMEM)
    uint32_t lane, bt, k;  // bt: lane column byte | image 0 page
    const uint8_t* skew_codes;
    const uint64_t* ids;
    uint32_t* gthr;
    uint32_t* pool_key;
    uint64_t* pool_id;
    uint32_t* mslot;   // this warp's stash for the item: key[32], pos[32] (SMEM)
    uint32_t* mbase;   // the item's stashes, 64 words per warp
    uint32_t* mcount;  // warps of the item done so far
    uint32_t nact;     // warps with a non-empty range in the item
};

// Offers the completed entries of two consecutive tiles at once: one
// threshold refresh and one vote per pair of tiles.
__device__ __forceinline__ void topk_offer2(WarpTopK& t, uint32_t ka, bool va, uint32_t pa, uint32_t kb, bool vb,
                                            uint32_t pb, uint32_t lane, uint32_t k, const uint64_t* __restrict__ ids,
                                            uint32_t* gthr_q, uint32_t* cta_thr) {
    t.g = min(t.g, *reinterpret_cast<volatile uint32_t*>(cta_thr));  // other warps of this item
    const uint32_t lim = min(t.thr, t.g);
    const bool passa = va && ka <= lim, passb = vb && kb <= lim;
    if (!__any_sync(0xffffffffu, passa || passb)) return;
    topk_insert(t, ka, passa, pa, lane, k, ids);
    topk_insert(t, kb, passb && kb <= t.thr, pb, lane, k, ids);
    if (t.thr < t.g) {
        if (lane == 0) {
            atomicMin(gthr_q, t.thr);
            atomicMin(cta_thr, t.thr);
        }
        t.g = t.thr;
    }
}

// This warp's tile range [a, e_end) of an item (empty when a >= e_end).
template <int W>
__device__ __forceinline__ void warp_range(const ItemSlot& sl, uint32_t warp, uint32_t& a, uint32_t& e_end) {
    const uint32_t ntile = sl.te - sl.tb;
    const uint32_t nw = min(uint32_t(W), (ntile + kMinWarpTiles - 1) / kMinWarpTiles);
    const uint32_t per = (ntile + nw - 1) / nw;
    a = sl.tb + warp * per;
    e_end = warp < nw ? min(sl.te, a + per) : a;
}

// Warps of an item that get a non-empty range (a < te) from warp_range.
template <int W>
__device__ __forceinline__ uint32_t warp_count(const ItemSlot& sl) {
    const uint32_t ntile = sl.te - sl.tb;
    const uint32_t nw = min(uint32_t(W), (ntile + kMinWarpTiles - 1) / kMinWarpTiles);
    const uint32_t per = (ntile + nw - 1) / nw;
    return min(nw, (ntile + per - 1) / per);
}

// Stash the warp's list of the item; the item's last warp merges the lists
// and publishes the item's top-k to its pool slot.
__device__ __forceinline__ void merge_publish(const ScanCtx& cx, const ItemSlot& sl, const WarpTopK& t,
                                              uint32_t* gthr_q) {
    const uint32_t lane = cx.lane, k = cx.k;
    const uint64_t* __restrict__ ids = cx.ids;
    // Stash this warp's list; the item's last warp merges the stashed lists
    // into the CTA's exact top-k of the item and publishes only that (k
    // entries per item reach the query's pool instead of k per warp).
    cx.mslot[lane] = lane < k ? t.key : 0xffffffffu;
    cx.mslot[32 + lane] = t.pos;
    __syncwarp();
    uint32_t arrived = 0;
    if (lane == 0) {
        __threadfence_block();
        arrived = atomicAdd(cx.mcount, 1u);
    }
    arrived = __shfl_sync(0xffffffffu, arrived, 0);
    if (arrived + 1 < cx.nact) return;
    __threadfence_block();
    if (lane == 0) *cx.mcount = 0;  // the buffer's next item starts from zero
    // k rounds of "smallest (key, id) among the list heads" (lane w < nact
    // owns warp w's list, sorted by (distance, chunk id))
    const uint32_t* ml = cx.mbase + lane * 64;
    const bool own = lane < cx.nact;
    uint32_t hi = 0;
    uint32_t hk = own ? ml[0] : 0xffffffffu, hp = own ? ml[32] : 0u;
    uint32_t rk = 0xffffffffu, rp = 0u, cnt = 0;
    for (uint32_t r = 0; r < k; ++r) {
        const uint32_t kmin = __reduce_min_sync(0xffffffffu, hk);
        if (kmin == 0xffffffffu) break;
        const unsigned tie = __ballot_sync(0xffffffffu, hk == kmin);
        int win = __ffs(tie) - 1;
        if (tie & (tie - 1)) {  // exact distance tie between lists: lowest chunk id first
            uint64_t id = hk == kmin ? ids[hp] : ~0ull;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const uint64_t oid = __shfl_xor_sync(0xffffffffu, id, o);
                id = oid < id ? oid : id;
            }
            win = __ffs(__ballot_sync(0xffffffffu, hk == kmin && ids[hp] == id)) - 1;
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
    if (cnt == k) {
        const uint32_t kth = __shfl_sync(0xffffffffu, rk, k - 1);
        if (lane == 0) atomicMin(gthr_q, kth);
    }
    // the item's fixed pool slot: k entries, unfilled ones as +inf sentinels
    if (lane < k) {
        const size_t o = size_t(sl.pslot) * k + lane;
        cx.pool_key[o] = lane < cnt ? ord_key(__uint_as_float(rk)) : 0xffffffffu;
        // the entry slot, not the chunk id: an id load here (a global round
        // trip) would fall on the item's last warp every item, and that warp
        // then lags the others by more each item (measured ~1.5 us per item
        // at config B); K4 translates the few survivors' slots to ids
        cx.pool_id[o] = lane < cnt ? uint64_t(rp) : ~0ull;
    }
}

// One consumer warp's share [a, e_end] of an item: tiles a..e_end inclusive
// (tile e_end holds the tails of the range's last entries) are loaded into
// registers one tile ahead (A, B alternate) and folded against the SMEM
// image; lane 0 keeps the next kPrefetch tiles requested into L2 (the
// producer requested each range's first tiles when it fetched the item).
// Completed entries of each pair of tiles are
// offered to the warp's exact top-k, which is finally merged with the item's
// other warps and published to the query's candidate pool.
// BUF: the image buffer (compile-time: its offset from image 0 is part of
// every gather's immediate).
template <int M, int BUF>
__device__ __forceinline__ void scan_range(const ScanCtx& cx, const ItemSlot& sl, uint32_t a, uint32_t e_end,
                                           const float* mk, const float* nk, uint32_t P) {
    constexpr uint32_t kTileBytes = 32u * M;
    const uint32_t lane = cx.lane, bt = cx.bt, k = cx.k;
    const uint64_t* __restrict__ ids = cx.ids;
    uint32_t* gthr_q = cx.gthr + sl.q;
    const unsigned char* tiles = cx.skew_codes + sl.tile_byte_off;
    const unsigned char* src_lane = tiles + lane * 16;
    // the query's shared threshold (other CTAs' k-th distances), read once
    // per range; the producer's snapshot from item fetch time bounds it too
    WarpTopK t{0xffffffffu, 0xffffffffu, 0xffffffffu, min(sl.thr, ld_relaxed(gthr_q))};
    uint4 A[M / 16], B[M / 16];
    load_tile<M>(A, src_lane, a);
    load_tile<M>(B, src_lane, a + 1);  // ranges have >= 2 tiles
    // L2 window: tiles [a + 2, pf) requested so far (the producer requested
    // [a, a + kHeadTiles) at item fetch)
    uint32_t pf = P ? min(a + uint32_t(kHeadTiles), e_end + 1) : e_end + 1;
    const uint32_t lbase = uint32_t(sl.lbase), len = sl.len;
    float cur = 0.0f, prev = 0.0f;
    for (uint32_t j = a;; j += 2) {
        // ---- tile j (registers A)
        skew_round<M, BUF * int(SkewSmem<M>::kImgStride)>(A, bt, cur, prev, mk, nk, std::make_integer_sequence<int, M>{});
        if (j + 2 <= e_end) load_tile<M>(A, src_lane, j + 2);
        const uint32_t ea = (j - 1) * kTileEntries + lane;  // entry completed in `prev`
        const uint32_t ka = __float_as_uint(prev);
        const bool va = j > a && ea < len;
        prev = cur;
        cur = 0.0f;
        if (j + 1 > e_end) {
            topk_offer2(t, ka, va, lbase + ea, 0xffffffffu, false, 0u, lane, k, ids, gthr_q, cx.cta_thr);
            break;
        }
        // ---- tile j + 1 (registers B)
        skew_round<M, BUF * int(SkewSmem<M>::kImgStride)>(B, bt, cur, prev, mk, nk, std::make_integer_sequence<int, M>{});
        if (j + 3 <= e_end) load_tile<M>(B, src_lane, j + 3);
        const uint32_t eb = j * kTileEntries + lane;
        const uint32_t kb = __float_as_uint(prev);
        const bool vb = eb < len;
        prev = cur;
        cur = 0.0f;
        // slide the L2 window two tiles (kPrefetch ahead of the loads)
        if (pf <= e_end && pf < j + 4 + P) {
            const uint32_t pe = min(pf + 2, e_end + 1);
            if (lane == 0) prefetch_l2(tiles + size_t(pf) * kTileBytes, (pe - pf) * kTileBytes);
            pf = pe;
        }
        topk_offer2(t, ka, va, lbase + ea, kb, vb, lbase + eb, lane, k, ids, gthr_q, cx.cta_thr);
        if (j + 2 > e_end) break;
    }
    merge_publish(cx, sl, t, gthr_q);
}

// Persistent, one CTA per SM, warp-specialised:
//  * producer warp (one lane): pulls work items {pair, tile_begin,
//    tile_end} (largest first), resolves the list's metadata and bulk-copies
//    the pair's compact table T[m][256] into the staging buffer (32
//    subquantizers per round);
//  * kExp expander warps: transpose the staged table into the conflict-free
//    image (4x4 register transposes walked diagonally, so every LDS.128 /
//    STS.128 is conflict-free) in one of two image buffers -- item i+1's
//    image is built while item i is scanned;
//  * kWarps consumer warps: each scans a contiguous tile range of the item
//    (scan_range), keeps an exact top-k (k <= 32) in registers by (distance,
//    chunk_id), prunes with a per-query threshold shared through global
//    memory (atomicMin on the k-th distance), and the item's last warp merges
//    the warps' lists into the item's pool slot.
// "Data ready" hand-offs are mbarriers; "slot free" hand-offs are named
// barriers (a waiting warp is descheduled, arriving warps do not wait).
// Candidates are held as (distance bits, entry slot); chunk ids are loaded
// only on an exact distance tie and when a list is published.
template <int M>
__global__ void __launch_bounds__(SkewSmem<M>::threads, 1)
    scan_skew_kernel(const uint4* __restrict__ items, const uint32_t* __restrict__ num_items,
                     uint32_t* __restrict__ cursor, const uint32_t* __restrict__ probe,
                     const uint32_t* __restrict__ list_len, const uint64_t* __restrict__ skew_off,
                     const uint8_t* __restrict__ skew_codes, const uint64_t* __restrict__ list_off,
                     const uint64_t* __restrict__ ids, const float* __restrict__ luts, uint32_t nprobe,
                     uint32_t k, uint32_t* __restrict__ gthr, uint32_t* __restrict__ pool_key,
                     uint64_t* __restrict__ pool_id, uint32_t l2_prefetch, uint32_t tail_od) {
    CT_BEGIN;
    using L = SkewSmem<M>;
    constexpr int W = L::W, NB = L::NB;
    constexpr int kExpWarps = SkewCfg<M>::kExp;
    constexpr uint32_t kStageBytes = L::kStage;
    constexpr uint32_t kHalves = M / 32;  // staging rounds per item (32 subquantizers each)
    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t base = smem_u32(smem);
    const uint32_t img_off = ((base + L::kGuard + 0xffffu) & ~0xffffu) - base;  // image 0, 64 KiB-aligned
    const bool in_pad = img_off >= L::kGuard + L::kStage + L::kTail;
    const uint32_t stage_off = in_pad ? 0u : img_off + L::kImgSpan;
    const uint32_t tail_off = stage_off + L::kStage;
    if ((in_pad ? img_off + L::kImgSpan : tail_off + L::kTail) > L::bytes) __trap();
    float* stage = reinterpret_cast<float*>(smem + stage_off);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + tail_off);
    uint64_t* img_full = bars;
    uint64_t* stg_full = bars + NB;
    ItemSlot* slots = reinterpret_cast<ItemSlot*>(smem + tail_off + 8 * L::nbars);  // [NB] image slots
    ItemSlot* stg_slot = slots + NB;                                                  // staging slot
    uint32_t* cta_thr = reinterpret_cast<uint32_t*>(stg_slot + 1);  // [NB]: the CTA's k-th distance per item
    uint32_t* mcount = cta_thr + NB;                                  // [NB]: merge arrivals per item
    uint32_t* mstash = mcount + NB;                                   // [NB][W][64]: warp lists of an item

    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NB; ++i) {
            mbar_init(img_full + i, kExpWarps);
            mcount[i] = 0;
        }
        mbar_init(stg_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();  // items, LUTs and thresholds come from the previous kernels
    CT_WAITED(4);
    const uint32_t total = *num_items;
#ifdef PRAG_K3_TRACE
    unsigned long long* tr = g_k3_trace + size_t(blockIdx.x) * kTraceSlots;
    uint32_t ntr = 1;
    if (threadIdx.x == 0) tr[0] = gtime();
#endif

    // Barrier 1 + b: consumers arrive when done with image buffer b,
    // expanders sync before overwriting it. Barrier 1 + NB: expanders arrive
    // when done with the staging buffer, the producer syncs before refilling.
    constexpr uint32_t kImgEmptyCount = uint32_t(W + kExpWarps) * 32;
    constexpr uint32_t kStgEmptyCount = uint32_t(kExpWarps + 1) * 32;
    constexpr uint32_t kStgBar = 1 + NB;
    if (warp == uint32_t(W)) {
        // ------------------------------------------------------ producer
        // The next item's index is normally reserved one item ahead (its
        // metadata loads overlap the staging wait); within the last tail_od
        // items of the queue it is reserved only once the staging buffer is
        // free, so a CTA does not hold a tail item it cannot start soon.
        uint32_t nx = 0;
        if (lane == 0) nx = atomicAdd(cursor, 1u);
        bool held = true;     // nx is a reserved index
        uint32_t round = 0;  // staging rounds issued (kHalves per item)
#ifdef PRAG_K3_TRACE
        uint32_t pit = 0;
#endif
        for (;;) {
            bool synced = false;  // staging-free barrier already passed this item
            if (!held) {
                if (round > 0) named_sync(kStgBar, kStgEmptyCount);
                synced = true;
                if (lane == 0) nx = atomicAdd(cursor, 1u);
            }
            ItemSlot sl{};
            sl.pair = kEndItem;
            held = true;
            if (lane == 0 && nx < total) {
                const uint4 w4 = items[nx];
                const uint32_t list = probe[w4.x];
                sl.pair = w4.x;
                sl.tb = w4.y;
                sl.te = w4.z;
                sl.len = list_len[list];
                sl.q = w4.x / nprobe;
                sl.tile_byte_off = skew_off[list] * (32u * M);
                sl.lbase = list_off[list];
                sl.thr = ld_relaxed(gthr + sl.q);
                sl.pslot = w4.w;
                if (total - nx > tail_od)
                    nx = atomicAdd(cursor, 1u);  // next item's index, fetched ahead
                else
                    held = false;
            }
            held = __shfl_sync(0xffffffffu, held ? 1u : 0u, 0) != 0;
            const uint32_t pair = __shfl_sync(0xffffffffu, sl.pair, 0);
#ifdef PRAG_K3_TRACE
            if (lane == 0 && pair != kEndItem) K3T2(0, pit, gtime());
#endif
            if (pair == kEndItem) {
                pdl_trigger();  // no more work items: let the pool selection launch
                if (round > 0 && !synced) named_sync(kStgBar, kStgEmptyCount);
                if (lane == 0) {
                    *stg_slot = sl;
                    mbar_arrive(stg_full);
                }
                CT_END(4);
                break;
            }
            {  // request the head of every consumer warp's range into L2 now, an
               // item or two before the consumers reach it
                ItemSlot r{};
                r.tb = __shfl_sync(0xffffffffu, sl.tb, 0);
                r.te = __shfl_sync(0xffffffffu, sl.te, 0);
                const uint64_t tbo = __shfl_sync(0xffffffffu, sl.tile_byte_off, 0);
                uint32_t wa, we;
                warp_range<W>(r, lane, wa, we);
                if (l2_prefetch && lane < uint32_t(W) && wa < we)
                    prefetch_l2(skew_codes + tbo + size_t(wa) * (32u * M), min(we - wa + 1, kHeadTiles) * (32u * M));
            }
            const unsigned char* src = reinterpret_cast<const unsigned char*>(luts) + size_t(pair) * M * 1024;
            for (uint32_t h = 0; h < kHalves; ++h, ++round) {
                if (round > 0 && !(h == 0 && synced)) named_sync(kStgBar, kStgEmptyCount);
                if (lane == 0) {
                    if (h == 0) *stg_slot = sl;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(stg_full, kStageBytes);
                    bulk_g2s(stage, src + h * kStageBytes, kStageBytes, stg_full);
#ifdef PRAG_K3_TRACE
                    if (h == 0) K3T2(1, pit, gtime());
#endif
                }
            }
#ifdef PRAG_K3_TRACE
            ++pit;
#endif
        }
        return;
    }
    if (warp > uint32_t(W)) {
        // ------------------------------------------------------ expanders
        const uint32_t ew = warp - W - 1;
        uint32_t round = 0;
        for (uint32_t i = 0;; ++i) {
            const uint32_t b = i % NB;
            mbar_wait(stg_full, round & 1u);
#ifdef PRAG_K3_TRACE
            if (ew == 0 && lane == 0) K3T2(2, i, gtime());
#endif
            const ItemSlot sl = *stg_slot;
            if (i >= uint32_t(NB)) named_sync(1 + b, kImgEmptyCount);  // consumers done with item i - NB
#ifdef PRAG_K3_TRACE
            if (ew == 0 && lane == 0) K3T2(3, i, gtime());
#endif
            if (sl.pair == kEndItem) {
                __syncwarp();
                if (lane == 0) {
                    if (ew == 0) {
                        slots[b] = sl;
                        cta_thr[b] = 0xffffffffu;
                    }
                    mbar_arrive(img_full + b);
                }
                CT_END(4);
                break;
            }
            float* img = reinterpret_cast<float*>(smem + img_off + b * L::kImgStride);
            for (uint32_t h = 0; h < kHalves; ++h, ++round) {
                if (h > 0) mbar_wait(stg_full, round & 1u);
                // 4x4 register transposes: lane L owns codes cb + 4L .. +3 and
                // walks the 8 groups of 4 subquantizers diagonally (group
                // (g + L) mod 8), so every LDS.128 (4 codes of one staged row)
                // and STS.128 (4 columns of one image row) is conflict-free;
                // units (code block of 128, subquantizer group step): 2 x 8,
                // dealt round-robin to the expander warps
#pragma unroll 2
                for (uint32_t u = ew; u < 16; u += kExpWarps) {
                    const uint32_t c4 = (u >> 3) * 128 + 4 * lane;
                    const uint32_t g = u & 7u;
                    const uint32_t sq0 = 4 * ((g + lane) & 7u);  // local subquantizer group
                    float4 v[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) v[r] = *reinterpret_cast<const float4*>(stage + (sq0 + r) * 256 + c4);
                    const float4 col[4] = {make_float4(v[0].x, v[1].x, v[2].x, v[3].x),
                                           make_float4(v[0].y, v[1].y, v[2].y, v[3].y),
                                           make_float4(v[0].z, v[1].z, v[2].z, v[3].z),
                                           make_float4(v[0].w, v[1].w, v[2].w, v[3].w)};
                    const uint32_t sq = 32 * h + sq0;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        float* row = img + (c4 + i) * 64;
                        if (M == 32) {  // column c = T[c mod 32]: columns sq and sq + 32
                            *reinterpret_cast<float4*>(row + sq) = col[i];
                            *reinterpret_cast<float4*>(row + sq + 32) = col[i];
                        } else {        // column c = T[c]; row 255's upper half also in the guard
                            *reinterpret_cast<float4*>(row + sq) = col[i];
                            if (c4 + i == 255 && h == 1) *reinterpret_cast<float4*>(img - 64 + sq) = col[i];
                        }
                    }
                }
                named_arrive(kStgBar, kStgEmptyCount);  // staging consumed
            }
            __syncwarp();
            if (lane == 0) {
                if (ew == 0) {
                    slots[b] = sl;
                    cta_thr[b] = 0xffffffffu;
                }
                mbar_arrive(img_full + b);
#ifdef PRAG_K3_TRACE
                if (ew == 0) K3T2(4, i, gtime());
#endif
            }
        }
        return;
    }

    // -------------------------------------------------------- consumers
    // lane's column byte 4 (31 - lane) (the step's column offset is in the
    // gather's immediate) and image 0's 64 KiB page in bytes 2-3
    const uint32_t bt = (31u - lane) * 4u | ((base + img_off) & 0xffff0000u);
    // step masks: {1, 0} where step s >= lane (the starting entry), {0, 1}
    // before (the finishing entry); one FFMA2 updates {cur, prev}.
    float mk[32], nk[32];
#pragma unroll
    for (int s = 0; s < 32; ++s) {
        mk[s] = (uint32_t(s) >= lane) ? 1.0f : 0.0f;
        nk[s] = (uint32_t(s) >= lane) ? 0.0f : 1.0f;
    }

    for (uint32_t i = 0;; ++i) {
        const uint32_t b = i % NB;
        mbar_wait(img_full + b, (i / NB) & 1u);
        const ItemSlot sl = slots[b];
#ifdef PRAG_K3_TRACE
        const unsigned long long t_item = gtime();
#endif
        if (sl.pair == kEndItem) {
#ifdef PRAG_K3_TRACE
            if (warp == 0 && lane == 0 && ntr < kTraceSlots) tr[ntr++] = t_item | (1ull << 63);
            if (warp == 0 && lane == 0) tr[kTraceSlots - 1] = ntr;
#endif
            CT_END(4);
            break;
        }
        uint32_t a, e_end;
        warp_range<W>(sl, warp, a, e_end);
        if (a < e_end) {
            uint32_t* mb = mstash + b * (W * 64);
            const ScanCtx cx{cta_thr + b, lane, bt, k, skew_codes, ids, gthr, pool_key, pool_id, mb + warp * 64,
                             mb, mcount + b, warp_count<W>(sl)};
            if (b == 0)
                scan_range<M, 0>(cx, sl, a, e_end, mk, nk, l2_prefetch);
            else
                scan_range<M, 1>(cx, sl, a, e_end, mk, nk, l2_prefetch);
        }
#ifdef PRAG_K3_TRACE
        if (warp == uint32_t(W) - 1 && lane == 0) K3T2(5, i, gtime());
        if (warp == 0 && lane == 0 && ntr + 3 < kTraceSlots) {
            tr[ntr++] = t_item;
            tr[ntr++] = gtime();
            tr[ntr++] = sl.te - sl.tb;
        }
#endif
        __syncwarp();
        named_arrive(1 + b, kImgEmptyCount);  // image buffer b is free
    }
}

}  // namespace

#ifdef PRAG_CHAIN_TRACE
CT_BIND_FN(ct_bind_skew)
#endif

#ifdef PRAG_K3_TRACE
extern "C" int prag_gpu_debug_k3_trace(unsigned long long* out, size_t n) {
    return cudaMemcpyFromSymbol(out, g_k3_trace, std::min(n, size_t(160 * kTraceSlots)) * 8) == cudaSuccess ? 0 : 3;
}
extern "C" int prag_gpu_debug_k3_trace2(unsigned long long* out, size_t n) {
    return cudaMemcpyFromSymbol(out, g_k3_trace2, std::min(n, size_t(160 * 6 * 32)) * 8) == cudaSuccess ? 0 : 3;
}
#endif

uint32_t skew_item_tiles(uint64_t est_tiles, uint32_t grid) {
    // enough items for ~per_cta per CTA, within [kMinItemTiles, kMaxItemTiles]
    // (PRAG_GPU_ITEMS_PER_CTA overrides the default of 1, best in tools/sweep_items.sh; tuning knob)
    const char* e = getenv("PRAG_GPU_ITEMS_PER_CTA");
    const long v = e ? atol(e) : 0;
    const uint64_t per_cta = uint64_t(v > 0 ? v : 1);
    uint64_t want = est_tiles / (uint64_t(grid) * per_cta + 1);
    uint32_t it = kMinItemTiles;
    while (it < kMaxItemTiles && uint64_t(it) * 2 <= want) it *= 2;
    return it;
}
uint32_t skew_min_item_tiles() { return kMinItemTiles; }
uint32_t skew_warps(uint32_t m) { return m == 32 ? SkewCfg<32>::kWarps : SkewCfg<64>::kWarps; }
size_t skew_lut_bytes(uint32_t m) { return size_t(m) * 1024; }  // compact T[m][256] per pair

static int check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("CUDA launch failed (") + what + "): " + cudaGetErrorString(e));
        return PRAG_GPU_CUDA;
    }
    return PRAG_GPU_OK;
}

int launch_lut_images(const DeviceIndex& ix, const float* queries, const uint32_t* probe, uint32_t nq,
                      uint32_t nprobe, float* luts, uint32_t it_tiles, uint64_t* scanned, uint4* items,
                      uint32_t* num_items, uint32_t* cursor, uint32_t* q_item_off, uint32_t* gthr,
                      uint32_t* pair_off, uint64_t item_cap, uint32_t scan_grid, cudaStream_t s) {
    const uint32_t npairs = nq * nprobe;
    // tail splitting (register planners only, nq * nprobe <= 2048): off by
    // default. Measured (tools/item_sweep.py, PRAG_GPU_SPLIT_ITEMS = 0 / 148 /
    // 296 / 592 split items): config C batch 1 at nprobe 128 / 256 within
    // +-1%, nprobe 64 -6%, config B nq 64 -3%. The K3 timeline
    // (tools/k3_trace.py) shows why: CTAs finish within ~8 us of each other
    // (p10-p90) already; the time goes to the fold itself (warp 0 busy 86% of
    // the span at config C batch 1), not to the last items.
    const char* se = getenv("PRAG_GPU_SPLIT_ITEMS");
    const uint32_t split = se ? uint32_t(atoi(se)) : 0u;
    const PlanArgs pa{it_tiles, split, scanned, items, num_items, cursor, q_item_off, gthr, pair_off, item_cap};
    // G table CTAs: two per SM of the search's SM budget with the planner
    // taking one of the slots, at most one per task
    const uint32_t ntasks = (npairs + kTaskPairs - 1) / kTaskPairs * ix.nsq;
    const uint32_t G = std::max<uint32_t>(1u, std::min<uint32_t>(2u * scan_grid - 1u, ntasks));
    const dim3 grid(G + 1);
#define PG_LUT(MM, SS)                                                                                          \
    PG_CUDA(launch_pdl(lut_tasks_kernel<MM, SS>, grid, dim3(256), 0, s, queries, ix.centroids, ix.codewordsT,   \
                       probe, ix.list_len, nq, nprobe, ix.d, ix.sub_dim, luts, pa))
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
                     const uint32_t* probe, const float* luts, uint32_t nprobe, uint32_t k, uint32_t* gthr,
                     uint32_t* pool_key, uint64_t* pool_id, int grid, cudaStream_t s) {
    // L2 prefetch distance in tiles (0: off); PRAG_GPU_L2_PREFETCH overrides (tuning knob)
    const char* pe = getenv("PRAG_GPU_L2_PREFETCH");
    const uint32_t l2pf = pe ? uint32_t(atoi(pe)) : uint32_t(ix.nsq == 32 ? SkewCfg<32>::kPrefetch : SkewCfg<64>::kPrefetch);
    // on-demand reservation of the queue's last 4 x grid items (0: always one
    // ahead). Measured (tools/r3_knobs*.sh, 0 / 148 / 296 / 592 / 1184 / all):
    // 592 best or tied on every config B / C row (config B nq 8, nprobe 64
    // -8%, nq 64, nprobe 16 -1.5%). PRAG_GPU_TAIL_ONDEMAND overrides (tuning knob).
    const char* te = getenv("PRAG_GPU_TAIL_ONDEMAND");
    const uint32_t tail_od = te ? uint32_t(atoi(te)) : 4u * uint32_t(grid);
    if (ix.nsq == 32) {
        const size_t smem = skew_smem_bytes<32>();
        PG_CUDA(ensure_smem(reinterpret_cast<const void*>(scan_skew_kernel<32>), int(smem)));
        PG_CUDA(launch_pdl(scan_skew_kernel<32>, dim3(grid), dim3(SkewSmem<32>::threads), smem, s, items, num_items,
                           cursor, probe, ix.list_len, ix.skew_off, ix.skew_codes, ix.list_off, ix.ids, luts, nprobe, k,
                           gthr, pool_key, pool_id, l2pf, tail_od));
    } else {
        const size_t smem = skew_smem_bytes<64>();
        PG_CUDA(ensure_smem(reinterpret_cast<const void*>(scan_skew_kernel<64>), int(smem)));
        PG_CUDA(launch_pdl(scan_skew_kernel<64>, dim3(grid), dim3(SkewSmem<64>::threads), smem, s, items, num_items,
                           cursor, probe, ix.list_len, ix.skew_off, ix.skew_codes, ix.list_off, ix.ids, luts, nprobe, k,
                           gthr, pool_key, pool_id, l2pf, tail_od));
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
                    // lane t's byte s lives in 16-byte chunk s/16 at chunk*512 + t*16 + s%16;
                    // m = 64 stores a tail byte (s < t) as code + 1 (see SkewSmem)
                    const uint8_t c = ok ? codes[e * m + byte] : 0;
                    tile[(s / 16) * 512 + t * 16 + (s % 16)] = (m == 64 && s < t) ? uint8_t(c + 1) : c;
                }
            }
        }
    }
}

}  // namespace pg
