// embed.cu -- query embedding on the device, the step
// that precedes search in LocalRetriever::retrieve (pipeline.hpp:227).
//
// prag::ChunkEmbedder::embed (tokendb.hpp:95-112) is a bag-of-tokens
// embedding: the double-precision sum of the fp32 unit vectors of the
// non-PAD tokens, in token order, divided by its L2 norm and rounded to fp32
// (e_0 for an all-PAD chunk). The token vectors (tokendb.hpp:63-80) come from
// SplitMix64 Box-Muller draws through libm log/cos/sqrt, which the GPU's libm
// does not reproduce to the last ulp, so they are computed here on the host,
// exactly as the reference does, for token ids [0, vocab) and kept in HBM.
// The kernel then reproduces the rest op for op (IEEE double add / mul /
// sqrt / div, FMA-free), so embeddings are bit-identical to the reference's.
#include <cmath>
#include <cstdint>
#include <memory>
#include <unordered_map>
#include <vector>

#include "internal.h"

struct prag_gpu_embedder {
    int device = 0;
    uint32_t d = 0, vocab = 0;
    uint64_t seed = 0;
    float* table = nullptr;  // [vocab][d] fp32 token unit vectors
    uint32_t* tok = nullptr; // staging for host token chunks
    float* out = nullptr;    // staging for host outputs
    size_t tok_cap = 0, out_cap = 0;
    float* extra = nullptr;  // per-call rows for token ids >= vocab (host tokens)
    size_t extra_cap = 0;    // floats
};

namespace pg {
namespace {

// common.hpp:33-64 (SplitMix64), :66-71 (hash_combine); host only.
struct Mix64 {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double next_gaussian() {
        double u1 = next_double();
        double u2 = next_double();
        while (u1 <= 0.0) u1 = next_double();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    }
};

uint64_t mix_combine(uint64_t a, uint64_t b) {
    uint64_t z = a + 0x9e3779b97f4a7c15ULL + (b << 6) + (b >> 2);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// token_unit_vector (tokendb.hpp:63-80)
void token_vector(uint32_t token, uint32_t d, uint64_t seed, float* out) {
    Mix64 rng{mix_combine(seed, token)};
    std::vector<double> v(d);
    double norm_sq = 0.0;
    for (uint32_t i = 0; i < d; ++i) {
        v[i] = rng.next_gaussian();
        norm_sq += v[i] * v[i];
    }
    const double norm = std::sqrt(norm_sq);
    if (norm < 1e-12) {
        for (uint32_t i = 0; i < d; ++i) out[i] = 0.0f;
        out[0] = 1.0f;
        return;
    }
    for (uint32_t i = 0; i < d; ++i) out[i] = static_cast<float>(v[i] / norm);
}

constexpr int kEmbThreads = 128;

// One CTA per chunk. Thread i accumulates dims i, i + 128, ... over the
// chunk's tokens in order (tokendb.hpp:99-103); one thread folds the squared
// norm sequentially over dims (:104-105); every thread divides (:110).
// Token rows: ids < vocab from the resident table, ids in [vocab, vocab +
// n_extra) from this call's extra rows (host-computed for ids the database
// vocabulary did not cover; the staged tokens are remapped to them).
__global__ void __launch_bounds__(kEmbThreads) embed_kernel(const float* __restrict__ table, uint32_t vocab, uint32_t d,
                                                            const float* __restrict__ extra, uint32_t n_extra,
                                                            const uint32_t* __restrict__ tokens, uint32_t m,
                                                            float* __restrict__ out, uint32_t* __restrict__ bad) {
    extern __shared__ double acc_s[];  // [d]
    __shared__ double norm_s;
    const uint32_t c = blockIdx.x, tid = threadIdx.x;
    const uint32_t* tk = tokens + size_t(c) * m;
    for (uint32_t i = tid; i < d; i += kEmbThreads) {
        double acc = 0.0;
        for (uint32_t t = 0; t < m; ++t) {
            const uint32_t tok = tk[t];
            if (tok == 0) continue;  // kPadToken (common.hpp:16)
            if (tok - vocab < n_extra) {  // (unsigned: false for tok < vocab)
                acc = __dadd_rn(acc, double(__ldg(extra + size_t(tok - vocab) * d + i)));
                continue;
            }
            if (tok >= vocab) {
                if (i == 0) atomicExch(bad, 1u);
                continue;
            }
            acc = __dadd_rn(acc, double(__ldg(table + size_t(tok) * d + i)));
        }
        acc_s[i] = acc;
    }
    __syncthreads();
    if (tid == 0) {
        double ns = 0.0;
        for (uint32_t i = 0; i < d; ++i) ns = __dadd_rn(ns, __dmul_rn(acc_s[i], acc_s[i]));
        norm_s = ns < 1e-24 ? -1.0 : __dsqrt_rn(ns);
    }
    __syncthreads();
    const double norm = norm_s;
    for (uint32_t i = tid; i < d; i += kEmbThreads)
        out[size_t(c) * d + i] = norm < 0.0 ? (i == 0 ? 1.0f : 0.0f) : __double2float_rn(__ddiv_rn(acc_s[i], norm));
}

bool dev_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace
}  // namespace pg

using namespace pg;

extern "C" {

int prag_gpu_embedder_create(uint32_t d, uint64_t seed, uint32_t vocab, int device, prag_gpu_embedder** out) {
    PG_API_BEGIN
    if (!out) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    *out = nullptr;
    if (d < 2) {  // tokendb.hpp:88
        set_error("ChunkEmbedder: d must be >= 2");
        return PRAG_GPU_CONFIG;
    }
    if (vocab < 1) {
        set_error("embedder: vocab must be >= 1");
        return PRAG_GPU_CONFIG;
    }
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        set_error("no CUDA device visible: the prag_gpu embedder has no CPU fallback");
        return PRAG_GPU_NO_DEVICE;
    }
    auto e = std::make_unique<prag_gpu_embedder>();
    e->device = device;
    e->d = d;
    e->vocab = vocab;
    e->seed = seed;
    std::vector<float> host(size_t(vocab) * d);
    for (uint32_t t = 0; t < vocab; ++t) token_vector(t, d, seed, host.data() + size_t(t) * d);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaError_t err = cudaMalloc(&e->table, host.size() * 4);
    if (err == cudaSuccess) err = cudaMemcpy(e->table, host.data(), host.size() * 4, cudaMemcpyHostToDevice);
    cudaSetDevice(prev);
    if (err != cudaSuccess) {
        cudaFree(e->table);
        set_error(std::string("CUDA error (embedder table): ") + cudaGetErrorString(err));
        return err == cudaErrorMemoryAllocation ? PRAG_GPU_OOM : PRAG_GPU_CUDA;
    }
    *out = e.release();
    return PRAG_GPU_OK;
    PG_API_END
}

void prag_gpu_embedder_free(prag_gpu_embedder* e) {
    if (!e) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(e->device);
    cudaDeviceSynchronize();
    cudaFree(e->table);
    cudaFree(e->tok);
    cudaFree(e->out);
    cudaFree(e->extra);
    cudaSetDevice(prev);
    delete e;
}

int prag_gpu_embed(prag_gpu_embedder* e, const uint32_t* tokens, uint32_t nchunks, uint32_t m, float* out,
                   void* stream) {
    PG_API_BEGIN
    if (!e || (!tokens && nchunks && m) || (!out && nchunks)) {
        set_error("null argument");
        return PRAG_GPU_CONFIG;
    }
    if (nchunks == 0) return PRAG_GPU_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(e->device);
    struct Restore {
        int dev;
        ~Restore() { cudaSetDevice(dev); }
    } restore{prev};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool tok_dev = dev_ptr(tokens), out_dev = dev_ptr(out);
    const size_t tok_n = size_t(nchunks) * m, out_n = size_t(nchunks) * e->d;
    if (e->tok_cap < tok_n + 1) {
        PG_CUDA(cudaStreamSynchronize(s));
        cudaFree(e->tok);
        e->tok = nullptr;
        e->tok_cap = 0;
        PG_CUDA(cudaMalloc(&e->tok, (tok_n + 1) * 4));
        e->tok_cap = tok_n + 1;
    }
    uint32_t* bad = e->tok + tok_n;  // error flag after the staged tokens
    const uint32_t* dtok = tokens;
    uint32_t n_extra = 0;
    if (!tok_dev) {
        // ChunkEmbedder::embed computes any token's vector on demand
        // (tokendb.hpp:63-80, :99-103): ids beyond the resident table get
        // their rows computed here for this call, so no id is out of range
        // and one request never fails the others embedded with it.
        std::unordered_map<uint32_t, uint32_t> slot;
        std::vector<uint32_t> staged;
        for (size_t i = 0; i < tok_n; ++i) {
            const uint32_t t = tokens[i];
            if (t < e->vocab) continue;
            if (staged.empty()) staged.assign(tokens, tokens + tok_n);
            auto it = slot.emplace(t, e->vocab + uint32_t(slot.size())).first;
            staged[i] = it->second;
        }
        n_extra = uint32_t(slot.size());
        if (n_extra) {
            if (uint64_t(e->vocab) + n_extra > 0xffffffffull) {
                set_error("embed: too many distinct token ids");
                return PRAG_GPU_CONFIG;
            }
            std::vector<float> rows(size_t(n_extra) * e->d);
            for (const auto& kv : slot) token_vector(kv.first, e->d, e->seed, rows.data() + size_t(kv.second - e->vocab) * e->d);
            if (e->extra_cap < rows.size()) {
                PG_CUDA(cudaStreamSynchronize(s));
                cudaFree(e->extra);
                e->extra = nullptr;
                e->extra_cap = 0;
                PG_CUDA(cudaMalloc(&e->extra, rows.size() * 4));
                e->extra_cap = rows.size();
            }
            // pageable sources: both copies have consumed their host buffers on return
            PG_CUDA(cudaMemcpyAsync(e->extra, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, s));
            PG_CUDA(cudaMemcpyAsync(e->tok, staged.data(), tok_n * 4, cudaMemcpyHostToDevice, s));
        } else {
            PG_CUDA(cudaMemcpyAsync(e->tok, tokens, tok_n * 4, cudaMemcpyHostToDevice, s));
        }
        dtok = e->tok;
    }
    float* dout = out;
    if (!out_dev) {
        if (e->out_cap < out_n) {
            PG_CUDA(cudaStreamSynchronize(s));
            cudaFree(e->out);
            e->out = nullptr;
            e->out_cap = 0;
            PG_CUDA(cudaMalloc(&e->out, out_n * 4));
            e->out_cap = out_n;
        }
        dout = e->out;
    }
    PG_CUDA(cudaMemsetAsync(bad, 0, 4, s));
    embed_kernel<<<nchunks, kEmbThreads, size_t(e->d) * 8, s>>>(e->table, e->vocab, e->d, e->extra, n_extra, dtok, m,
                                                                 dout, bad);
    PG_CUDA(cudaGetLastError());
    if (!out_dev || !tok_dev) {
        uint32_t hbad = 0;
        if (!out_dev) PG_CUDA(cudaMemcpyAsync(out, dout, out_n * 4, cudaMemcpyDeviceToHost, s));
        PG_CUDA(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s));
        PG_CUDA(cudaStreamSynchronize(s));
        if (hbad) {
            set_error("embed: token id >= embedder vocab");
            return PRAG_GPU_CONFIG;
        }
    }
    return PRAG_GPU_OK;
    PG_API_END
}

}  // extern "C"
