// decode_stub.cu -- the generator side of the config-E harness (BASELINE.json
// configs[4]): a memory-bound stand-in for one RETRO
// decode step, so retrieval on a side stream can be overlapped with -- and
// contend for HBM with -- real GPU work. It plays the role of the
// reference's SyntheticGenerator (generator.hpp:220-252), whose per-token
// cost is affine in position: here a GEMV over the model's fp32 weights
// (constant term; PAPER.md:347/703 RETRO 582M -> ~2.3 GB per token) plus a
// read of the KV cache of every earlier position (the linear term).
#include <cstdint>

#include "internal.h"

namespace pg {
namespace {

// y[r] = sum_j W[r][j] * x[j]  (cols % 4 == 0), one warp per row, grid-stride,
// then a pass over the KV cache folded into a data-dependent sink so the
// reads stay live. Exactly one 1024-thread CTA per SM on `gridDim.x` SMs (its
// dynamic shared-memory request, more than half an SM's, keeps a second one
// off the SM): with fewer CTAs than SMs the remaining SMs stay free for
// retrieval kernels on a side stream (config E: PipeRAG overlap without the
// decode holding every SM).
constexpr int kPartThreads = 1024;
constexpr size_t kPartSmem = 120 * 1024;

__global__ void __launch_bounds__(kPartThreads, 1) decode_part_kernel(const float4* __restrict__ w, uint64_t rows,
                                                                      uint32_t cols4, const float4* __restrict__ x,
                                                                      float* __restrict__ y,
                                                                      const float4* __restrict__ kv, uint64_t kv4) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * kPartThreads + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * kPartThreads) >> 5;
    for (uint64_t r = warp; r < rows; r += nwarps) {
        const float4* row = w + r * cols4;
        float acc = 0.0f;
        for (uint32_t j = lane; j < cols4; j += 32) {
            const float4 a = __ldcs(row + j);
            const float4 b = __ldg(x + j);
            acc += a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) y[r] = acc;
    }
    float s = 0.0f;
    for (uint64_t i = uint64_t(blockIdx.x) * kPartThreads + threadIdx.x; i < kv4;
         i += uint64_t(gridDim.x) * kPartThreads) {
        const float4 v = __ldcs(kv + i);
        s += v.x + v.y + v.z + v.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && s == 1234.5678f) y[rows] = s;
}

}  // namespace
}  // namespace pg

extern "C" int prag_gpu_synthetic_decode_sms(const float* weights, uint64_t rows, uint32_t cols, const float* x,
                                             float* y, const float* kv, uint64_t kv_floats, uint32_t sms,
                                             void* stream) {
    using namespace pg;
    if (!weights || !x || !y || cols % 4 != 0 || (kv_floats && !kv) || kv_floats % 4 != 0 || sms == 0) {
        set_error("synthetic_decode_sms: bad arguments (cols, kv_floats multiples of 4; sms >= 1)");
        return PRAG_GPU_CONFIG;
    }
    int dev = 0, all = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&all, cudaDevAttrMultiProcessorCount, dev);
    if (int(sms) > all) sms = uint32_t(all);
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(decode_part_kernel), kPartSmem);
    if (e == cudaSuccess) {
        decode_part_kernel<<<sms, kPartThreads, kPartSmem, static_cast<cudaStream_t>(stream)>>>(
            reinterpret_cast<const float4*>(weights), rows, cols / 4, reinterpret_cast<const float4*>(x), y,
            reinterpret_cast<const float4*>(kv), kv_floats / 4);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) {
        set_error(std::string("CUDA launch failed (synthetic_decode_sms): ") + cudaGetErrorString(e));
        return PRAG_GPU_CUDA;
    }
    return PRAG_GPU_OK;
}

extern "C" int prag_gpu_synthetic_decode(const float* weights, uint64_t rows, uint32_t cols, const float* x, float* y,
                                         const float* kv, uint64_t kv_floats, void* stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return prag_gpu_synthetic_decode_sms(weights, rows, cols, x, y, kv, kv_floats, uint32_t(sms), stream);
}
