// train.cu -- index build on the device: prag::train_index
// (annindex.hpp:164-241) with its k-means (annindex.hpp:62-130), reproduced
// bit for bit. Build is off the query path; it feeds it (PRAGIX01 files and
// in-HBM indexes for configs B-D) and reuses the same arithmetic primitive
// (common.hpp:73-80, sequential FMA-free fp32 fold).
//
// What is parallel and what is not (every result is identical to the
// reference's sequential code):
//  * nearest_kernel: all (point, centroid) squared distances of one k-means
//    assignment, final IVF assignment or PQ encoding, as a register-tiled SIMT
//    "GEMM" whose inner product is the reference's fold (sub, mul, add in
//    dimension order, no contraction); per point the first minimum with the
//    reference's `dsq < best` rule (best starts at FLT_MAX) via a
//    lexicographic (distance, index) reduction.
//  * kmeans++ seeding: min-distance update across the grid, then ONE thread
//    per problem runs the double prefix sum `total += min_dist[i]`
//    (annindex.hpp:80-83) in point order -- a rounding-order dependent chain
//    that cannot be reassociated -- and the pick is a parallel lower_bound on
//    the stored prefix (the reference's second loop recomputes the same
//    prefix, annindex.hpp:87-91).
//  * Lloyd update: members of each cluster in point order (stable radix sort
//    of (cluster, point)), one thread per (cluster, dimension) folding the
//    double sums in that order (annindex.hpp:113-117), IEEE division and
//    rounding to fp32 (:128); empty clusters re-seeded sequentially in
//    cluster order from the first farthest point (:119-126).
//  * PQ codebooks: the nsq subspace k-means problems run batched.
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.h"

namespace pg {
namespace {

// ------------------------------------------------------------ SplitMix64
// common.hpp:33-53 (integer part only: bit-identical on host and device).
__host__ __device__ __forceinline__ uint64_t sm_next(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ double sm_next_double(uint64_t& s) {
    return static_cast<double>(sm_next(s) >> 11) * 0x1.0p-53;
}
// common.hpp:66-71
uint64_t hash_combine_h(uint64_t a, uint64_t b) {
    uint64_t z = a + 0x9e3779b97f4a7c15ULL + (b << 6) + (b >> 2);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ------------------------------------------------------- nearest_kernel
// Point sources. Layout 0: row-major rows (the caller's vectors), optionally
// gathered through `rows` and optionally minus the assigned coarse centroid
// (the residual of annindex.hpp:201 computed on the fly, same fp32 sub).
// Layout 1: transposed training sets [problem][dim][np] (coalesced loads).
struct PointSrc {
    const float* base = nullptr;
    uint64_t stride = 0;        // layout 0: row stride; layout 1: np
    uint64_t prob_step = 0;     // per problem: layout 0 column offset, layout 1 element offset
    const uint32_t* rows = nullptr;
    const float* sub_cent = nullptr;
    const uint32_t* sub_assign = nullptr;
    int layout = 0;
};

struct NearestArgs {
    PointSrc p;
    uint64_t np = 0;
    uint32_t dim = 0, K = 0;
    const float* cents = nullptr;   // per problem [K][dim]
    uint64_t cent_step = 0;
    uint32_t* out_c = nullptr;      // [problem][np] (out_step apart)
    float* out_d = nullptr;
    uint64_t out_step = 0;
    uint8_t* out_code = nullptr;    // [np][code_stride], column = problem
    uint32_t code_stride = 0;
};

constexpr int kTP = 64, kTC = 128, kKC = 16, kNT = 256;

// (c0 - w)^2, (c1 - w)^2 as FADD2 + FMUL2: |fl(c - w)| == |fl(w - c)|, so the
// squares equal the reference's diff*diff exactly; the sums stay scalar FADDs
// so nothing can contract into an FMA.
__device__ __forceinline__ void subsq2(float c0, float c1, float w, float& s0, float& s1) {
    unsigned long long out;
    asm("{.reg .b64 A, B, D;\n"
        " mov.b64 A, {%1, %2};\n"
        " mov.b64 B, {%3, %3};\n"
        " sub.rn.f32x2 D, A, B;\n"
        " mul.rn.f32x2 %0, D, D;}"
        : "=l"(out)
        : "f"(c0), "f"(c1), "f"(w));
    s0 = __uint_as_float(uint32_t(out));
    s1 = __uint_as_float(uint32_t(out >> 32));
}

__device__ __forceinline__ float load_point(const NearestArgs& a, uint32_t b, uint64_t i, uint32_t j) {
    const PointSrc& s = a.p;
    if (s.layout == 1) return s.base[b * s.prob_step + uint64_t(j) * s.stride + i];
    const uint64_t row = s.rows ? s.rows[i] : i;
    const uint64_t col = b * s.prob_step + j;
    float v = s.base[row * s.stride + col];
    if (s.sub_cent) v = __fsub_rn(v, s.sub_cent[uint64_t(s.sub_assign[row]) * s.stride + col]);
    return v;
}

// One CTA: 64 points x all K centroids, 128 centroids per tile, dimensions in
// chunks of 16 staged in SMEM (zero padding is exact: acc + (0-0)^2 == acc).
// Thread (ty, tx) owns points ty*4..+3 and centroids tx*8..+7 of a tile.
__global__ void __launch_bounds__(kNT) nearest_kernel(NearestArgs a) {
    __shared__ __align__(16) float Ps[kKC][kTP];
    __shared__ __align__(16) float Cs[kKC][kTC];
    __shared__ float red_d[16][kTP];
    __shared__ uint32_t red_c[16][kTP];
    const uint32_t b = blockIdx.y;
    const uint64_t p0 = uint64_t(blockIdx.x) * kTP;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const float* cents = a.cents + b * a.cent_step;
    float best[4];
    uint32_t bc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        best[i] = FLT_MAX;
        bc[i] = 0xffffffffu;
    }
    for (uint32_t c0 = 0; c0 < a.K; c0 += kTC) {
        float acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
        for (uint32_t k0 = 0; k0 < a.dim; k0 += kKC) {
            __syncthreads();
            for (int e = tid; e < kKC * kTP; e += kNT) {
                int p, k;
                if (a.p.layout == 1) {
                    k = e / kTP;
                    p = e % kTP;
                } else {
                    p = e / kKC;
                    k = e % kKC;
                }
                const uint64_t i = p0 + p;
                const uint32_t j = k0 + k;
                Ps[k][p] = (i < a.np && j < a.dim) ? load_point(a, b, i, j) : 0.0f;
            }
            for (int e = tid; e < kKC * kTC; e += kNT) {
                const int c = e / kKC, k = e % kKC;
                const uint32_t cc = c0 + c, j = k0 + k;
                Cs[k][c] = (cc < a.K && j < a.dim) ? cents[uint64_t(cc) * a.dim + j] : 0.0f;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kKC; ++k) {
                const float4 pv = *reinterpret_cast<const float4*>(&Ps[k][ty * 4]);
                const float4 ca = *reinterpret_cast<const float4*>(&Cs[k][tx * 8]);
                const float4 cb = *reinterpret_cast<const float4*>(&Cs[k][tx * 8 + 4]);
                const float pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    float s[8];
                    subsq2(ca.x, ca.y, pw[i], s[0], s[1]);
                    subsq2(ca.z, ca.w, pw[i], s[2], s[3]);
                    subsq2(cb.x, cb.y, pw[i], s[4], s[5]);
                    subsq2(cb.z, cb.w, pw[i], s[6], s[7]);
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = __fadd_rn(acc[i][j], s[j]);
                }
            }
        }
        // ascending centroid order within the thread: first minimum kept
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t c = c0 + tx * 8 + j;
                if (c < a.K && acc[i][j] < best[i]) {
                    best[i] = acc[i][j];
                    bc[i] = c;
                }
            }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        red_d[tx][ty * 4 + i] = best[i];
        red_c[tx][ty * 4 + i] = bc[i];
    }
    __syncthreads();
    if (tid < kTP) {
        float d = red_d[0][tid];
        uint32_t c = red_c[0][tid];
        for (int t = 1; t < 16; ++t) {
            const float d2 = red_d[t][tid];
            const uint32_t c2 = red_c[t][tid];
            if (c2 != 0xffffffffu && (c == 0xffffffffu || d2 < d || (d2 == d && c2 < c))) {
                d = d2;
                c = c2;
            }
        }
        if (c == 0xffffffffu) {  // no dsq < FLT_MAX: best_c stays 0 (annindex.hpp:101-102)
            c = 0;
            d = FLT_MAX;
        }
        const uint64_t i = p0 + tid;
        if (i < a.np) {
            if (a.out_c) a.out_c[b * a.out_step + i] = c;
            if (a.out_d) a.out_d[b * a.out_step + i] = d;
            if (a.out_code) a.out_code[i * a.code_stride + b] = uint8_t(c);
        }
    }
}

// ----------------------------------------------------------- k-means++
// min_dist[i] = min(min_dist[i], squared_l2(point i, last centroid))
// (annindex.hpp:79-82).
__global__ void pp_update_kernel(const float* __restrict__ PT, uint64_t np, uint32_t dim,
                                 const float* __restrict__ C, uint64_t cent_step, uint32_t t,
                                 float* __restrict__ md) {
    const uint32_t b = blockIdx.y;
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= np) return;
    const float* c = C + b * cent_step + uint64_t(t - 1) * dim;
    const float* p = PT + uint64_t(b) * dim * np + i;
    float acc = 0.0f;
    for (uint32_t j = 0; j < dim; ++j) {
        const float d = __fsub_rn(p[uint64_t(j) * np], __ldg(c + j));
        acc = __fadd_rn(acc, __fmul_rn(d, d));
    }
    float& m = md[b * np + i];
    if (acc < m) m = acc;
}

constexpr int kPickThreads = 1024, kPickChunk = 8192;

// One CTA per problem. Thread 0 folds the double prefix in point order; the
// block then finds the first prefix >= r (prefixes are non-decreasing), and
// copies the picked point into centroid t (annindex.hpp:83-95).
__global__ void __launch_bounds__(kPickThreads) pp_pick_kernel(const float* __restrict__ md, double* __restrict__ pref,
                                                               uint64_t np, uint64_t* __restrict__ rng,
                                                               uint32_t t, const float* __restrict__ PT,
                                                               uint32_t dim, float* __restrict__ C, uint64_t cent_step) {
    __shared__ float buf[kPickChunk];
    __shared__ double r_s;
    __shared__ int mode_s;
    __shared__ unsigned long long pick_s;
    const uint32_t b = blockIdx.x;
    const float* m = md + b * np;
    double* pr = pref + b * np;
    double s = 0.0;
    for (uint64_t base = 0; base < np; base += kPickChunk) {
        const uint32_t len = np - base < uint64_t(kPickChunk) ? uint32_t(np - base) : uint32_t(kPickChunk);
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < len; e += kPickThreads) buf[e] = m[base + e];
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll 8
            for (uint32_t e = 0; e < len; ++e) {
                s = __dadd_rn(s, double(buf[e]));
                pr[base + e] = s;
            }
        }
    }
    if (threadIdx.x == 0) {
        uint64_t st = rng[b];
        if (s > 0.0) {
            r_s = __dmul_rn(sm_next_double(st), s);
            mode_s = 1;
            pick_s = ~0ull;
        } else {
            mode_s = 0;
            pick_s = sm_next(st) % np;
        }
        rng[b] = st;
    }
    __syncthreads();
    if (mode_s == 1) {
        const double r = r_s;
        unsigned long long first = ~0ull;
        for (uint64_t i = threadIdx.x; i < np; i += kPickThreads)
            if (pr[i] >= r) {
                first = i;
                break;
            }
        if (first != ~0ull) atomicMin(&pick_s, first);
        __syncthreads();
        if (threadIdx.x == 0 && pick_s == ~0ull) pick_s = 0;  // loop never broke: pick stays 0
        __syncthreads();
    }
    const uint64_t pick = pick_s;
    float* dst = C + b * cent_step + uint64_t(t) * dim;
    for (uint32_t j = threadIdx.x; j < dim; j += kPickThreads) dst[j] = PT[uint64_t(b) * dim * np + uint64_t(j) * np + pick];
}

// first = rng.next_below(n); centroid 0 = that point (annindex.hpp:74-76)
__global__ void pp_first_kernel(uint64_t np, uint64_t* rng, const float* PT, uint32_t dim, float* C, uint64_t cent_step,
                                float* md) {
    const uint32_t b = blockIdx.x;
    __shared__ unsigned long long first_s;
    if (threadIdx.x == 0) {
        uint64_t st = rng[b];
        first_s = sm_next(st) % np;
        rng[b] = st;
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < dim; j += blockDim.x)
        C[b * cent_step + j] = PT[uint64_t(b) * dim * np + uint64_t(j) * np + first_s];
    for (uint64_t i = threadIdx.x; i < np; i += blockDim.x) md[b * np + i] = FLT_MAX;
}

// ---------------------------------------------------------------- Lloyd
__global__ void key_kernel(const uint32_t* __restrict__ assign, uint64_t np, uint32_t K, uint32_t B,
                           uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t* __restrict__ counts) {
    const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= np * B) return;
    const uint32_t b = uint32_t(e / np);
    const uint32_t key = b * K + assign[e];
    keys[e] = key;
    vals[e] = uint32_t(e - uint64_t(b) * np);
    atomicAdd(counts + key, 1u);
}

// centroid[c][j] = float(sum_{members in point order} double(x[j]) / count)
__global__ void centroid_kernel(const float* __restrict__ PT, uint64_t np, uint32_t dim, uint32_t K, uint32_t B,
                                const uint32_t* __restrict__ counts, const uint32_t* __restrict__ offs,
                                const uint32_t* __restrict__ members, float* __restrict__ C, uint64_t cent_step) {
    const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= uint64_t(B) * K * dim) return;
    const uint32_t j = uint32_t(e % dim);
    const uint64_t bc = e / dim;
    const uint32_t b = uint32_t(bc / K), c = uint32_t(bc % K);
    const uint32_t cnt = counts[bc];
    if (cnt == 0) return;
    const uint32_t* mem = members + offs[bc];
    const float* col = PT + uint64_t(b) * dim * np + uint64_t(j) * np;
    double s = 0.0;
    for (uint32_t q = 0; q < cnt; ++q) s = __dadd_rn(s, double(col[mem[q]]));
    C[b * cent_step + uint64_t(c) * dim + j] = __double2float_rn(__ddiv_rn(s, double(cnt)));
}

// Empty clusters, in cluster order: the first point with the largest
// assign_dist (strict >, from -1) becomes the centroid and its assign_dist
// drops to 0 (annindex.hpp:119-126).
__global__ void __launch_bounds__(1024) reseed_kernel(const float* __restrict__ PT, uint64_t np, uint32_t dim,
                                                      uint32_t K, const uint32_t* __restrict__ counts,
                                                      float* __restrict__ adist, float* __restrict__ C,
                                                      uint64_t cent_step) {
    __shared__ float rv[32];
    __shared__ unsigned long long ri[32];
    __shared__ unsigned long long far_s;
    const uint32_t b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    float* ad = adist + b * np;
    for (uint32_t c0 = 0; c0 < K; c0 += 1024) {
        const uint32_t c = c0 + tid;
        const bool empty = c < K && counts[uint64_t(b) * K + c] == 0;
        if (!__syncthreads_or(empty)) continue;
        for (uint32_t cc = c0; cc < min(K, c0 + 1024); ++cc) {
            if (counts[uint64_t(b) * K + cc] != 0) continue;
            float bv = -1.0f;
            unsigned long long bi = 0;
            for (uint64_t i = tid; i < np; i += 1024)
                if (ad[i] > bv) {
                    bv = ad[i];
                    bi = i;
                }
            for (int o = 16; o; o >>= 1) {
                const float ov = __shfl_down_sync(0xffffffffu, bv, o);
                const unsigned long long oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            if (lane == 0) {
                rv[wid] = bv;
                ri[wid] = bi;
            }
            __syncthreads();
            if (tid == 0) {
                float v = rv[0];
                unsigned long long ix = ri[0];
                for (int w = 1; w < 32; ++w)
                    if (rv[w] > v || (rv[w] == v && ri[w] < ix)) {
                        v = rv[w];
                        ix = ri[w];
                    }
                far_s = ix;
                ad[ix] = 0.0f;
            }
            __syncthreads();
            const uint64_t far = far_s;
            for (uint32_t j = tid; j < dim; j += 1024)
                C[b * cent_step + uint64_t(cc) * dim + j] = PT[uint64_t(b) * dim * np + uint64_t(j) * np + far];
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------- gathers
// PT[b][j][i] = x[sample[i]][b*dim + j] (minus centroid[assign[sample[i]]])
__global__ void gather_t_kernel(const float* __restrict__ X, uint32_t d, const uint64_t* __restrict__ sample, uint64_t ns,
                                uint32_t dim, uint32_t B, const float* __restrict__ cents,
                                const uint32_t* __restrict__ assign, float* __restrict__ PT) {
    const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= ns * d) return;
    const uint64_t i = e % ns;
    const uint32_t col = uint32_t(e / ns);  // b*dim + j
    const uint64_t row = sample[i];
    float v = X[row * d + col];
    if (cents) v = __fsub_rn(v, cents[uint64_t(assign[row]) * d + col]);
    const uint32_t b = col / dim, j = col % dim;
    PT[uint64_t(b) * dim * ns + uint64_t(j) * ns + i] = v;
    (void)B;
}

__global__ void iota_u32_kernel(uint32_t* v, uint64_t n) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = uint32_t(i);
}

__global__ void count_kernel(const uint32_t* __restrict__ assign, uint64_t n, uint32_t* __restrict__ counts) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) atomicAdd(counts + assign[i], 1u);
}

__global__ void widen_kernel(const uint32_t* __restrict__ in, uint64_t n, uint64_t* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[i];
}

__global__ void offsets_kernel(const uint32_t* __restrict__ counts, uint32_t nlist, uint64_t* __restrict__ off) {
    // single thread: nlist <= a few 1e5, off the hot path
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        uint64_t s = 0;
        off[0] = 0;
        for (uint32_t l = 0; l < nlist; ++l) {
            s += counts[l];
            off[l + 1] = s;
        }
    }
}

// ------------------------------------------------------------ buffers
struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { cudaFree(p); }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

#define PG_ALLOC(buf, bytes) PG_CUDA(cudaMalloc(&(buf).p, std::max<size_t>(size_t(bytes), 16)))

inline uint32_t blocks_for(uint64_t n, uint32_t t) { return uint32_t((n + t - 1) / t); }

int launch_nearest(const NearestArgs& a, uint32_t B, cudaStream_t s) {
    if (a.np == 0) return PRAG_GPU_OK;
    const uint64_t gx = (a.np + kTP - 1) / kTP;
    if (gx > 0x7fffffffull || B > 65535) {
        set_error("train: grid too large");
        return PRAG_GPU_CONFIG;
    }
    nearest_kernel<<<dim3(uint32_t(gx), B), kNT, 0, s>>>(a);
    PG_CUDA(cudaGetLastError());
    return PRAG_GPU_OK;
}

// Batched k-means (annindex.hpp:64-130): B problems of np points of `dim`
// dims, transposed PT [B][dim][np]; C [B][K][dim] out.
int kmeans_batched(const float* PT, uint32_t B, uint64_t np, uint32_t dim, uint32_t K,
                   const std::vector<uint64_t>& seeds, int iterations, float* C, cudaStream_t s) {
    if (np < K) {
        set_error("kmeans: fewer points than clusters");
        return PRAG_GPU_CONFIG;
    }
    if (np > 0xffffffffull || uint64_t(B) * K > 0xffffffffull) {
        set_error("train: k-means problem too large (np must be < 2^32)");
        return PRAG_GPU_CONFIG;
    }
    const uint64_t cstep = uint64_t(K) * dim;
    DevBuf rng, md, pref;
    PG_ALLOC(rng, B * 8);
    PG_ALLOC(md, np * B * 4);
    PG_ALLOC(pref, np * B * 8);
    PG_CUDA(cudaMemcpyAsync(rng.p, seeds.data(), B * 8, cudaMemcpyHostToDevice, s));
    pp_first_kernel<<<B, 256, 0, s>>>(np, rng.as<uint64_t>(), PT, dim, C, cstep, md.as<float>());
    PG_CUDA(cudaGetLastError());
    for (uint32_t t = 1; t < K; ++t) {
        pp_update_kernel<<<dim3(blocks_for(np, 256), B), 256, 0, s>>>(PT, np, dim, C, cstep, t, md.as<float>());
        pp_pick_kernel<<<B, kPickThreads, 0, s>>>(md.as<float>(), pref.as<double>(), np, rng.as<uint64_t>(), t, PT,
                                                  dim, C, cstep);
    }
    PG_CUDA(cudaGetLastError());
    if (iterations <= 0) return PRAG_GPU_OK;

    const uint64_t ne = np * B;
    const uint32_t nkeys = B * K;
    DevBuf assign, adist, keys, vals, keys2, members, counts, offs, tmp;
    PG_ALLOC(assign, ne * 4);
    PG_ALLOC(adist, ne * 4);
    PG_ALLOC(keys, ne * 4);
    PG_ALLOC(vals, ne * 4);
    PG_ALLOC(keys2, ne * 4);
    PG_ALLOC(members, ne * 4);
    PG_ALLOC(counts, (nkeys + 1) * 4);
    PG_ALLOC(offs, (nkeys + 1) * 4);
    int end_bit = 1;
    while (end_bit < 32 && (uint64_t(1) << end_bit) < nkeys) ++end_bit;
    size_t sort_bytes = 0, scan_bytes = 0;
    PG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                            vals.as<uint32_t>(), members.as<uint32_t>(), int(ne), 0, end_bit, s));
    PG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts.as<uint32_t>(), offs.as<uint32_t>(),
                                          int(nkeys) + 1, s));
    PG_ALLOC(tmp, std::max(sort_bytes, scan_bytes));
    NearestArgs na;
    na.p.base = PT;
    na.p.layout = 1;
    na.p.stride = np;
    na.p.prob_step = np * dim;
    na.np = np;
    na.dim = dim;
    na.K = K;
    na.cents = C;
    na.cent_step = cstep;
    na.out_c = assign.as<uint32_t>();
    na.out_d = adist.as<float>();
    na.out_step = np;
    for (int it = 0; it < iterations; ++it) {
        PG_TRY(launch_nearest(na, B, s));
        PG_CUDA(cudaMemsetAsync(counts.p, 0, (nkeys + 1) * 4, s));
        key_kernel<<<blocks_for(ne, 256), 256, 0, s>>>(assign.as<uint32_t>(), np, K, B, keys.as<uint32_t>(),
                                                        vals.as<uint32_t>(), counts.as<uint32_t>());
        size_t sb = sort_bytes;
        PG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, sb, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                                vals.as<uint32_t>(), members.as<uint32_t>(), int(ne), 0, end_bit, s));
        size_t cb = scan_bytes;
        PG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, cb, counts.as<uint32_t>(), offs.as<uint32_t>(), int(nkeys) + 1, s));
        centroid_kernel<<<blocks_for(uint64_t(nkeys) * dim, 256), 256, 0, s>>>(
            PT, np, dim, K, B, counts.as<uint32_t>(), offs.as<uint32_t>(), members.as<uint32_t>(), C, cstep);
        reseed_kernel<<<B, 1024, 0, s>>>(PT, np, dim, K, counts.as<uint32_t>(), adist.as<float>(), C, cstep);
        PG_CUDA(cudaGetLastError());
    }
    return PRAG_GPU_OK;
}

// training_sample (annindex.hpp:134-145): partial Fisher-Yates over a virtual
// iota, SplitMix64(seed ^ 0x5a5a) -- host, O(cap).
std::vector<uint64_t> training_sample(uint64_t n, uint64_t cap, uint64_t seed) {
    std::vector<uint64_t> out;
    if (n <= cap) {
        out.resize(n);
        for (uint64_t i = 0; i < n; ++i) out[i] = i;
        return out;
    }
    std::unordered_map<uint64_t, uint64_t> moved;
    auto at = [&](uint64_t x) {
        auto it = moved.find(x);
        return it == moved.end() ? x : it->second;
    };
    uint64_t st = seed;
    out.resize(cap);
    for (uint64_t i = 0; i < cap; ++i) {
        const uint64_t j = i + sm_next(st) % (n - i);
        const uint64_t vi = at(i), vj = at(j);
        moved[i] = vj;
        moved[j] = vi;
        out[i] = vj;
    }
    return out;
}

bool dev_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace
}  // namespace pg

using namespace pg;

extern "C" {

int prag_gpu_train_index(const float* vectors, uint64_t n, uint32_t d, const prag_gpu_train_params* params,
                         int device, float* centroids, float* codewords, uint64_t* list_off, uint64_t* ids,
                         uint8_t* codes) {
    PG_API_BEGIN
    if (!params || (!vectors && n)) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    if (n == 0) {
        set_error("train_index: empty embedding set");
        return PRAG_GPU_CONFIG;
    }
    if (d == 0) {
        set_error("train_index: d must be >= 1");
        return PRAG_GPU_CONFIG;
    }
    const uint32_t nlist = params->nlist;
    if (nlist == 0) {
        set_error("train_index: nlist must be >= 1");
        return PRAG_GPU_CONFIG;
    }
    if (n < nlist) {
        set_error("train_index: nlist exceeds number of vectors");
        return PRAG_GPU_CONFIG;
    }
    const uint32_t nsq = params->n_subquantizers ? params->n_subquantizers : std::max(1u, d / 4);
    if (d % nsq != 0) {
        set_error("train_index: d not divisible by n_subquantizers");
        return PRAG_GPU_CONFIG;
    }
    if (n > 0xffffffffull) {
        set_error("train_index: the device trainer takes n < 2^32 vectors");
        return PRAG_GPU_CONFIG;
    }
    if (!centroids || !codewords || !list_off || !ids || !codes) {
        set_error("null output buffer");
        return PRAG_GPU_CONFIG;
    }
    const uint32_t sub = d / nsq;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        set_error("no CUDA device visible: the prag_gpu trainer has no CPU fallback");
        return PRAG_GPU_NO_DEVICE;
    }
    if (device < 0 || device >= ndev) {
        set_error("CUDA device out of range");
        return PRAG_GPU_CONFIG;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    struct Restore {
        int dev;
        ~Restore() { cudaSetDevice(dev); }
    } restore{prev};
    cudaStream_t s;
    PG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamFree {
        cudaStream_t s;
        ~StreamFree() {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    } sfree{s};

    // vectors on the device
    DevBuf xbuf;
    const float* X = vectors;
    if (!dev_ptr(vectors)) {
        PG_ALLOC(xbuf, n * d * 4);
        PG_CUDA(cudaMemcpyAsync(xbuf.p, vectors, n * d * 4, cudaMemcpyHostToDevice, s));
        X = xbuf.as<float>();
    }
    // training sample (annindex.hpp:178-180)
    const std::vector<uint64_t> sample = training_sample(n, params->train_sample_cap, params->seed ^ 0x5a5a);
    const uint64_t ns = sample.size();
    DevBuf samp, PT, C;
    PG_ALLOC(samp, ns * 8);
    PG_CUDA(cudaMemcpyAsync(samp.p, sample.data(), ns * 8, cudaMemcpyHostToDevice, s));
    PG_ALLOC(PT, ns * d * 4);
    PG_ALLOC(C, uint64_t(nlist) * d * 4);
    gather_t_kernel<<<blocks_for(ns * d, 256), 256, 0, s>>>(X, d, samp.as<uint64_t>(), ns, d, 1, nullptr, nullptr,
                                                             PT.as<float>());
    PG_CUDA(cudaGetLastError());
    // coarse centroids (annindex.hpp:186)
    PG_TRY(kmeans_batched(PT.as<float>(), 1, ns, d, nlist, {params->seed}, params->kmeans_iterations, C.as<float>(), s));

    // final assignment of every vector (annindex.hpp:195-202)
    DevBuf assign;
    PG_ALLOC(assign, n * 4);
    {
        NearestArgs na;
        na.p.base = X;
        na.p.layout = 0;
        na.p.stride = d;
        na.np = n;
        na.dim = d;
        na.K = nlist;
        na.cents = C.as<float>();
        na.out_c = assign.as<uint32_t>();
        PG_TRY(launch_nearest(na, 1, s));
    }
    // PQ codebooks on the sample residuals (annindex.hpp:209-218)
    const uint32_t pq_clusters = uint32_t(std::min<uint64_t>(256, n));
    const uint32_t clusters = uint32_t(std::min<uint64_t>(pq_clusters, ns));
    DevBuf RT, W, words;
    PG_ALLOC(RT, ns * d * 4);
    gather_t_kernel<<<blocks_for(ns * d, 256), 256, 0, s>>>(X, d, samp.as<uint64_t>(), ns, sub, nsq, C.as<float>(),
                                                             assign.as<uint32_t>(), RT.as<float>());
    PG_CUDA(cudaGetLastError());
    PG_ALLOC(W, uint64_t(nsq) * clusters * sub * 4);
    std::vector<uint64_t> seeds(nsq);
    for (uint32_t q = 0; q < nsq; ++q) seeds[q] = hash_combine_h(params->seed, q + 1);
    PG_TRY(kmeans_batched(RT.as<float>(), nsq, ns, sub, clusters, seeds, params->kmeans_iterations, W.as<float>(), s));
    // [nsq][256][sub], unused tail codes zero (annindex.hpp:217)
    PG_ALLOC(words, uint64_t(nsq) * 256 * sub * 4);
    PG_CUDA(cudaMemsetAsync(words.p, 0, uint64_t(nsq) * 256 * sub * 4, s));
    PG_CUDA(cudaMemcpy2DAsync(words.p, 256ull * sub * 4, W.p, uint64_t(clusters) * sub * 4, uint64_t(clusters) * sub * 4,
                              nsq, cudaMemcpyDeviceToDevice, s));

    // postings: entries of each list in vector order (annindex.hpp:222-238)
    DevBuf counts, off, keys2, vals, order, tmp, codes_d, ids_d;
    PG_ALLOC(counts, uint64_t(nlist) * 4);
    PG_ALLOC(off, (uint64_t(nlist) + 1) * 8);
    PG_ALLOC(keys2, n * 4);
    PG_ALLOC(vals, n * 4);
    PG_ALLOC(order, n * 4);
    PG_CUDA(cudaMemsetAsync(counts.p, 0, uint64_t(nlist) * 4, s));
    count_kernel<<<blocks_for(n, 256), 256, 0, s>>>(assign.as<uint32_t>(), n, counts.as<uint32_t>());
    offsets_kernel<<<1, 1, 0, s>>>(counts.as<uint32_t>(), nlist, off.as<uint64_t>());
    iota_u32_kernel<<<blocks_for(n, 256), 256, 0, s>>>(vals.as<uint32_t>(), n);
    PG_CUDA(cudaGetLastError());
    int end_bit = 1;
    while (end_bit < 32 && (uint64_t(1) << end_bit) < nlist) ++end_bit;
    size_t sort_bytes = 0;
    PG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, assign.as<uint32_t>(), keys2.as<uint32_t>(),
                                            vals.as<uint32_t>(), order.as<uint32_t>(), int(n), 0, end_bit, s));
    PG_ALLOC(tmp, sort_bytes);
    PG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, sort_bytes, assign.as<uint32_t>(), keys2.as<uint32_t>(),
                                            vals.as<uint32_t>(), order.as<uint32_t>(), int(n), 0, end_bit, s));
    // encode in list-major order (annindex.hpp:225-236)
    const bool codes_dev = dev_ptr(codes), ids_dev = dev_ptr(ids);
    uint8_t* codes_out = codes;
    if (!codes_dev) {
        PG_ALLOC(codes_d, n * nsq);
        codes_out = codes_d.as<uint8_t>();
    }
    {
        NearestArgs na;
        na.p.base = X;
        na.p.layout = 0;
        na.p.stride = d;
        na.p.prob_step = sub;
        na.p.rows = order.as<uint32_t>();
        na.p.sub_cent = C.as<float>();
        na.p.sub_assign = assign.as<uint32_t>();
        na.np = n;
        na.dim = sub;
        na.K = pq_clusters;
        na.cents = words.as<float>();
        na.cent_step = 256ull * sub;
        na.out_code = codes_out;
        na.code_stride = nsq;
        PG_TRY(launch_nearest(na, nsq, s));
    }
    uint64_t* ids_out = ids;
    if (!ids_dev) {
        PG_ALLOC(ids_d, n * 8);
        ids_out = ids_d.as<uint64_t>();
    }
    widen_kernel<<<blocks_for(n, 256), 256, 0, s>>>(order.as<uint32_t>(), n, ids_out);
    PG_CUDA(cudaGetLastError());
    const cudaMemcpyKind kind = cudaMemcpyDefault;
    PG_CUDA(cudaMemcpyAsync(centroids, C.p, uint64_t(nlist) * d * 4, kind, s));
    PG_CUDA(cudaMemcpyAsync(codewords, words.p, uint64_t(nsq) * 256 * sub * 4, kind, s));
    PG_CUDA(cudaMemcpyAsync(list_off, off.p, (uint64_t(nlist) + 1) * 8, kind, s));
    if (!ids_dev) PG_CUDA(cudaMemcpyAsync(ids, ids_out, n * 8, kind, s));
    if (!codes_dev) PG_CUDA(cudaMemcpyAsync(codes, codes_out, n * nsq, kind, s));
    PG_CUDA(cudaStreamSynchronize(s));
    return PRAG_GPU_OK;
    PG_API_END
}

}  // extern "C"
