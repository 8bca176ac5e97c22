// skew_common.cuh -- device helpers shared by the list-scan kernels (K3
// scan_skew_kernel, scan_skew.cu) and the batch-1 single-launch search
// (batch1.cu): async-copy / mbarrier wrappers, the lane-skewed ADC fold over
// the conflict-free SMEM table image, and the exact warp top-k.
//
// The fold and image layout are described in scan_skew.cu (file comment and
// SkewSmem); every add is the reference's sequential fp32 fold
// (annindex.hpp:300-302), ties ordered by (distance, chunk_id)
// (annindex.hpp:54-60).
#pragma once

#include <cstdint>
#include <utility>

#include "internal.h"

namespace pg {
namespace skew {

constexpr uint32_t kTileEntries = 32;

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

// Blocking wait: try_wait with a suspend-time hint, so a waiting warp is
// descheduled until the phase completes instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra LAB_WAIT;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase), "r"(0x989680u)
        : "memory");
}


__device__ __forceinline__ void named_sync(uint32_t id, uint32_t count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(uint32_t id, uint32_t count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
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


// LUT gather: 32-bit shared::cta address (the PRMT result) plus a
// compile-time offset.
template <int IMM>
__device__ __forceinline__ float lds_lut(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(IMM));
    return v;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Streaming 16-byte load of code bytes: read once per search, kept out of L1.
__device__ __forceinline__ uint4 ldg_codes(const unsigned char* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// One step of the skewed fold: lane's code byte S -> table column, gather,
// and the masked {cur, prev} update (steps >= 32 always belong to `cur`).
// OFF: byte offset of the gathered image from the one whose 64 KiB page is
// in bt (compile-time, so it folds into the LDS immediate).
template <int M, int OFF, int S>
__device__ __forceinline__ void skew_step(const uint4* v, uint32_t bt, float& cur, float& prev, const float* mk,
                                          const float* nk) {
    constexpr int IMM = (M == 32 ? 4 * (S + 1) : 4 * (S - 31)) + OFF;
    const uint4 c = v[S >> 4];
    const uint32_t w = ((S >> 2) & 3) == 0 ? c.x : ((S >> 2) & 3) == 1 ? c.y : ((S >> 2) & 3) == 2 ? c.z : c.w;
    // bytes: 0 = lane column (bt byte 0), 1 = code byte S & 3, 2-3 = image page (bt bytes 2-3)
    const uint32_t addr = __byte_perm(w, bt, 0x7604u | (uint32_t(S & 3) << 4));
    const float t = lds_lut<IMM>(addr);
    if constexpr (S < 32) {
        fma2_bcast(cur, prev, t, mk[S], nk[S]);
    } else {
        cur = __fadd_rn(cur, t);
    }
}

template <int M, int OFF, int... S>
__device__ __forceinline__ void skew_round(const uint4* v, uint32_t bt, float& cur, float& prev, const float* mk,
                                           const float* nk, std::integer_sequence<int, S...>) {
    (skew_step<M, OFF, S>(v, bt, cur, prev, mk, nk), ...);
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}


// Exact warp top-k (k <= 32): lane i holds the i-th (distance bits, entry
// slot) by (distance, chunk_id) (annindex.hpp:55-58); `thr` is the k-th key
// (0xffffffff until the list is full) and `g` the warp's view of the query's
// shared threshold. Chunk ids are read only on an exact distance tie.
struct WarpTopK {
    uint32_t key, pos, thr, g;
};

// (key, entry slot) order, used by the batched insertion below
__device__ __forceinline__ bool kp_less(uint32_t ka, uint32_t pa, uint32_t kb, uint32_t pb) {
    return ka < kb || (ka == kb && pa < pb);
}

// One compare-exchange step of a 32-lane bitonic network: the lower lane of
// each (lane, lane ^ stride) pair keeps the smaller (key, slot) when `asc`.
__device__ __forceinline__ void kp_cas(uint32_t& key, uint32_t& pos, uint32_t lane, uint32_t stride, bool asc) {
    const uint32_t ok = __shfl_xor_sync(0xffffffffu, key, stride);
    const uint32_t op = __shfl_xor_sync(0xffffffffu, pos, stride);
    const bool keep_small = ((lane & stride) == 0) == asc;
    if (keep_small == kp_less(ok, op, key, pos)) {
        key = ok;
        pos = op;
    }
}

// Batched insertion of the passing lanes (>= kBatchInsert of them): sort them
// across the warp (bitonic, by (key, slot)), merge with the sorted list
// (elementwise minimum against the reversed candidates, then a bitonic
// merge), keep the smallest 32. Orders ties by entry slot, not chunk id, so
// when the new first k + 1 hold an exact distance tie the list is restored
// and the exact one-at-a-time insertion runs instead (returns false).
#ifndef PRAG_BATCH_INSERT
#define PRAG_BATCH_INSERT 4
#endif
constexpr int kBatchInsert = PRAG_BATCH_INSERT;
__device__ __forceinline__ bool topk_insert_batch(WarpTopK& t, uint32_t key, bool pass, uint32_t mypos, uint32_t lane,
                                                  uint32_t k) {
    uint32_t ck = pass ? key : 0xffffffffu, cp = pass ? mypos : 0xffffffffu;
#pragma unroll
    for (uint32_t size = 2; size <= 32; size <<= 1)
#pragma unroll
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) kp_cas(ck, cp, lane, stride, (lane & size) == 0);
    const uint32_t rk = __shfl_sync(0xffffffffu, ck, 31 - lane), rp = __shfl_sync(0xffffffffu, cp, 31 - lane);
    uint32_t mk = t.key, mp = t.pos;
    if (kp_less(rk, rp, mk, mp)) {
        mk = rk;
        mp = rp;
    }
#pragma unroll
    for (uint32_t stride = 16; stride > 0; stride >>= 1) kp_cas(mk, mp, lane, stride, true);
    const uint32_t nk = __shfl_down_sync(0xffffffffu, mk, 1);
    if (__any_sync(0xffffffffu, lane < k && lane < 31 && mk == nk && mk != 0xffffffffu)) return false;
    t.key = mk;
    t.pos = mp;
    t.thr = __shfl_sync(0xffffffffu, t.key, k - 1);
    return true;
}

// Inserts the lanes' candidates that pass (rare after the first tiles; many
// at once go through the batched merge).
__device__ __forceinline__ void topk_insert(WarpTopK& t, uint32_t key, bool pass, uint32_t mypos, uint32_t lane,
                                            uint32_t k, const uint64_t* __restrict__ ids) {
    unsigned bal = __ballot_sync(0xffffffffu, pass);
    if (__popc(bal) >= kBatchInsert && topk_insert_batch(t, key, pass, mypos, lane, k)) return;
    while (bal) {
        const int src = __ffs(bal) - 1;
        bal &= bal - 1;
        const uint32_t ck = __shfl_sync(0xffffffffu, key, src);
        const uint32_t cp = __shfl_sync(0xffffffffu, mypos, src);
        if (ck > t.thr) continue;  // threshold tightened by an earlier insertion
        bool gt = t.key > ck;      // lanes whose element sorts after the candidate
        if (__any_sync(0xffffffffu, t.key == ck)) {  // exact distance tie: compare ids
            const uint64_t cid = ids[cp];
            const uint64_t mid = t.key == ck ? ids[t.pos] : 0ull;
            gt = gt || (t.key == ck && mid > cid);
        }
        const unsigned gm = __ballot_sync(0xffffffffu, gt);
        const int pos = gm ? __ffs(gm) - 1 : 32;
        if (pos < int(k)) {
            const uint32_t uk = __shfl_up_sync(0xffffffffu, t.key, 1);
            const uint32_t up = __shfl_up_sync(0xffffffffu, t.pos, 1);
            if (int(lane) > pos) {
                t.key = uk;
                t.pos = up;
            } else if (int(lane) == pos) {
                t.key = ck;
                t.pos = cp;
            }
            t.thr = __shfl_sync(0xffffffffu, t.key, k - 1);
        }
    }
}


template <int M>
__device__ __forceinline__ void load_tile(uint4 (&v)[M / 16], const unsigned char* src_lane, uint32_t j) {
#pragma unroll
    for (int c = 0; c < M / 16; ++c) v[c] = ldg_codes(src_lane + size_t(j) * (32u * M) + c * 512);
}



}  // namespace skew
}  // namespace pg
