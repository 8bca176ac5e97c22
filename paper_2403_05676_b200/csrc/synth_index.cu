// synth_index.cu -- config-D fixture builder (BASELINE.json configs[3],
// SURVEY.md 7.3 item 8 / 8d "D: a synthetic PQ index"): an IVF-PQ index of up
// to a few billion entries built directly in HBM, for the m = 32 / 64 fast
// path. Index build is not the query hot path; this exists
// because a 1B-entry PRAGIX01 file (~72 GB) and the reference's AoS in-memory
// index (~115 GB) cannot be staged through host memory here.
//
// A shard (prag_gpu_index_synthetic_shard) holds only its lists, each entry
// at its global position g, so its codes and chunk ids equal the full index's.
// Given centroids [nlist][d] and codewords [nsq][256][d/nsq] (the caller's,
// e.g. trained elsewhere), list sizes follow a log-normal skew drawn from
// SplitMix64 on the host; entry g (global, list-major) has chunk id g and
// PQ code bytes taken from W_i = splitmix_finalize(seed + 8 g + i):
// byte b = (W_{b/8} >> 8 (b%8)) & 0xff. The codes are written straight into
// the lane-skewed tile layout K3 reads; there is no plain [entry][m] copy, so
// such an index serves k <= 32 (the fast path) only.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <utility>
#include <vector>

#include "internal.h"

namespace pg {
namespace {

__host__ __device__ __forceinline__ uint64_t fin64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t code_byte(uint64_t seed, uint64_t g, uint32_t b) {
    const uint64_t w = fin64(seed + 8 * g + (b >> 3) + 0x9e3779b97f4a7c15ULL);
    return uint32_t(w >> (8 * (b & 7))) & 0xffu;
}

// One thread per (tile, lane): the lane's m bytes of the tile in fold-step
// order (scan_skew.cu build_skew_layout, on the device).
template <int M>
__global__ void synth_skew_kernel(const uint64_t* __restrict__ gbase, const uint64_t* __restrict__ rlen,
                                  const uint64_t* __restrict__ skew_off,
                                  uint32_t nlist, uint64_t seed, uint8_t* __restrict__ out, uint64_t ntiles) {
    const uint64_t gt = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t tile = gt >> 5;
    const uint32_t t = uint32_t(gt & 31);
    if (tile >= ntiles) return;
    // list of this tile: binary search in skew_off
    uint32_t lo = 0, hi = nlist;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (skew_off[mid] <= tile) lo = mid; else hi = mid;
    }
    const uint32_t l = lo;
    const uint64_t j = tile - skew_off[l];
    const uint64_t base = gbase[l], len = rlen[l];  // global position of entry 0, resident length
    uint8_t* dst = out + tile * (32ull * M);
#pragma unroll 4
    for (uint32_t s = 0; s < uint32_t(M); ++s) {
        uint64_t e;
        uint32_t byte;
        bool ok;
        if (s >= t) {
            e = j * 32 + t;
            byte = s - t;
            ok = e < len;
        } else {
            e = (j - 1) * 32 + t;
            byte = s - t + M;
            ok = j >= 1 && e < len;
        }
        const uint8_t c = ok ? uint8_t(code_byte(seed, base + e, byte)) : uint8_t(0);
        // m = 64: a tail byte (s < t) is stored as code + 1 (scan_skew.cu SkewSmem)
        dst[(s / 16) * 512 + t * 16 + (s % 16)] = (M == 64 && s < t) ? uint8_t(c + 1) : c;
    }
}

// ids of the padded list-major slots: chunk id g for real entries, ~0 pads
__global__ void synth_ids_kernel(const uint64_t* __restrict__ gbase, const uint64_t* __restrict__ rlen,
                                 const uint64_t* __restrict__ pad_off,
                                 uint32_t nlist, uint64_t* __restrict__ ids, uint64_t npadded) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= npadded) return;
    uint32_t lo = 0, hi = nlist;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (pad_off[mid] <= i) lo = mid; else hi = mid;
    }
    const uint64_t e = i - pad_off[lo];
    ids[i] = e < rlen[lo] ? gbase[lo] + e : ~0ull;
}

}  // namespace

// Host: log-normal list sizes summing to ntotal (largest-remainder rounding).
void synth_list_sizes(uint32_t nlist, uint64_t ntotal, uint64_t seed, double sigma, std::vector<uint64_t>& sizes) {
    std::vector<double> w(nlist);
    double sum = 0.0;
    uint64_t st = seed ^ 0x5bd1e995ULL;
    for (uint32_t l = 0; l < nlist; ++l) {
        auto u = [&]() { return double(fin64(st += 0x9e3779b97f4a7c15ULL) >> 11) * 0x1.0p-53; };
        double u1 = u(), u2 = u();
        while (u1 <= 0.0) u1 = u();
        const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
        w[l] = std::exp(sigma * z);
        sum += w[l];
    }
    sizes.assign(nlist, 0);
    uint64_t used = 0;
    std::vector<std::pair<double, uint32_t>> rem(nlist);
    for (uint32_t l = 0; l < nlist; ++l) {
        const double x = double(ntotal) * w[l] / sum;
        sizes[l] = uint64_t(x);
        used += sizes[l];
        rem[l] = {x - double(sizes[l]), l};
    }
    std::sort(rem.begin(), rem.end(), [](auto& a, auto& b) { return a.first > b.first || (a.first == b.first && a.second < b.second); });
    for (uint64_t i = 0; used < ntotal; ++i, ++used) ++sizes[rem[i % nlist].second];
}

int launch_synth_codes(uint32_t m, const uint64_t* gbase, const uint64_t* rlen, const uint64_t* skew_off, uint32_t nlist,
                       uint64_t seed, uint8_t* out, uint64_t ntiles, uint64_t* ids, const uint64_t* pad_off,
                       uint64_t npadded) {
    const uint64_t threads = ntiles * 32;
    const uint32_t blocks = uint32_t((threads + 255) / 256);
    if (m == 32)
        synth_skew_kernel<32><<<blocks, 256>>>(gbase, rlen, skew_off, nlist, seed, out, ntiles);
    else
        synth_skew_kernel<64><<<blocks, 256>>>(gbase, rlen, skew_off, nlist, seed, out, ntiles);
    PG_CUDA(cudaGetLastError());
    synth_ids_kernel<<<uint32_t((npadded + 255) / 256), 256>>>(gbase, rlen, pad_off, nlist, ids, npadded);
    PG_CUDA(cudaGetLastError());
    PG_CUDA(cudaDeviceSynchronize());
    return PRAG_GPU_OK;
}

}  // namespace pg
