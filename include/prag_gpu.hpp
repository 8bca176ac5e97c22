// prag_gpu.hpp -- C++ face of the B200 IVF-PQ retrieval path.
//
// Header-only wrapper over the C ABI in prag_gpu.h that gives the reference's
// C++ shapes back to a C++ host:
//
//   prag::gpu::Index           owns an HBM-resident index
//                              (replaces IvfIndex + PqCodebook, annindex.hpp:16-33)
//   prag::gpu::search(...)     prag::search (annindex.hpp:262-315), one query
//   prag::gpu::search_batch    the same for nq queries in one launch sequence
//   prag::gpu::calibrate_retrieval / select_nprobe
//                              perfmodel.hpp:92-117 / :148-157 fed by the GPU
//   prag::gpu::GpuRetriever    drop-in for prag::LocalRetriever
//                              (pipeline.hpp:213-249), compiled only when the
//                              reference's own headers are on the include
//                              path (the integrator's tree).
//
// Errors: status codes become exceptions. CONFIG -> prag::ConfigError and
// FORMAT -> prag::FormatError when the reference's common.hpp is included,
// otherwise prag::gpu::ConfigError / FormatError (both std::runtime_error,
// like common.hpp:23-29). Everything else -> prag::gpu::Error.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "prag_gpu.h"

#if defined(__has_include)
#if __has_include(<prag/pipeline.hpp>) && !defined(PRAG_GPU_NO_REFERENCE)
#include <prag/annindex.hpp>
#include <prag/perfmodel.hpp>
#include <prag/pipeline.hpp>
#define PRAG_GPU_HAVE_REFERENCE 1
#endif
#endif

namespace prag {
namespace gpu {

struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#ifdef PRAG_GPU_HAVE_REFERENCE
using ConfigError = ::prag::ConfigError;
using FormatError = ::prag::FormatError;
#else
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct FormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#endif

inline void check(int rc) {
    if (rc == PRAG_GPU_OK) return;
    std::string msg = prag_gpu_last_error();
    if (rc == PRAG_GPU_CONFIG) throw ConfigError(msg);
    if (rc == PRAG_GPU_FORMAT) throw FormatError(msg);
    throw Error(rc, msg);
}

// annindex.hpp:35-50 shapes (own copies so the header also works without the
// reference tree; with it, GpuRetriever converts to the reference types).
struct SearchParams {
    std::uint32_t nprobe = 1;
    std::uint32_t k = 2;
    bool exact_rerank = false;
};
struct ScoredId {
    std::uint64_t chunk_id = 0;
    float distance = 0.0f;
};
struct SearchResult {
    std::vector<ScoredId> neighbors;  // ascending distance, ties by lower id
    std::uint64_t scanned_vectors = 0;
    std::uint32_t scanned_lists = 0;
};
struct RetrievalPerfModel {  // perfmodel.hpp:19-26
    double slope_s = 0.0;
    double intercept_s = 0.0;
    double fit_residual_s = 0.0;
    bool clamped = false;
    double predict(std::uint32_t nprobe) const { return slope_s * nprobe + intercept_s; }
};

class Index {
public:
    // prag::load_index (annindex.hpp:361-411) straight into HBM of `device`.
    static Index load(const std::string& pragix01_path, int device = 0) {
        prag_gpu_index* h = nullptr;
        check(prag_gpu_index_load(pragix01_path.c_str(), device, &h));
        return Index(h);
    }
    // One list-sharded slice: rank's LPT share of the lists.
    static Index load_shard(const std::string& pragix01_path, int rank, int world, int device) {
        prag_gpu_index* h = nullptr;
        check(prag_gpu_index_load_shard(pragix01_path.c_str(), device, rank, world, &h));
        return Index(h);
    }
    // List-sharded over several GPUs of this process: LPT
    // placement, per-shard K1-K4 on each device, merge on devices[0] reading
    // the shards' top-k over NVLink. Usable wherever an Index is.
    static Index load_sharded(const std::string& pragix01_path, const std::vector<int>& devices) {
        prag_gpu_index* h = nullptr;
        check(prag_gpu_index_load_sharded(pragix01_path.c_str(), devices.data(), int(devices.size()), &h));
        return Index(h);
    }
    static Index from_host_sharded(std::uint32_t nlist, std::uint32_t d, std::uint32_t nsq, const float* centroids,
                                   const float* codewords, const std::uint64_t* list_off, const std::uint64_t* ids,
                                   const std::uint8_t* codes, const std::vector<int>& devices) {
        prag_gpu_index* h = nullptr;
        check(prag_gpu_index_from_host_sharded(nlist, d, nsq, centroids, codewords, list_off, ids, codes,
                                               devices.data(), int(devices.size()), &h));
        return Index(h);
    }
    // Flat host arrays in the reference's logical layout (see prag_gpu.h).
    static Index from_host(std::uint32_t nlist, std::uint32_t d, std::uint32_t nsq, const float* centroids,
                           const float* codewords, const std::uint64_t* list_off, const std::uint64_t* ids,
                           const std::uint8_t* codes, int device = 0) {
        prag_gpu_index* h = nullptr;
        check(prag_gpu_index_from_host(nlist, d, nsq, centroids, codewords, list_off, ids, codes, device, &h));
        return Index(h);
    }
#ifdef PRAG_GPU_HAVE_REFERENCE
    // The reference's in-memory objects (e.g. straight from train_index):
    // AoS postings are de-interleaved into the SoA arrays the ABI takes.
    static Index from_reference(const ::prag::IvfIndex& index, const ::prag::PqCodebook& cb, int device = 0) {
        return from_reference(index, cb, std::vector<int>{device});
    }
    // devices.size() > 1: list-sharded over those devices (see load_sharded)
    static Index from_reference(const ::prag::IvfIndex& index, const ::prag::PqCodebook& cb,
                                const std::vector<int>& devices) {
        const std::uint32_t nl = index.nlist, d = index.d, m = cb.n_subquantizers, sub = cb.sub_dim;
        std::vector<float> cent(std::size_t(nl) * d), words(std::size_t(m) * 256 * sub);
        for (std::uint32_t l = 0; l < nl; ++l)
            for (std::uint32_t j = 0; j < d; ++j) cent[std::size_t(l) * d + j] = index.centroids[l][j];
        for (std::uint32_t s = 0; s < m; ++s)
            for (std::uint32_t c = 0; c < 256; ++c)
                for (std::uint32_t j = 0; j < sub; ++j)
                    words[(std::size_t(s) * 256 + c) * sub + j] = cb.codewords[s][c][j];
        std::vector<std::uint64_t> off(std::size_t(nl) + 1, 0), ids;
        std::vector<std::uint8_t> codes;
        for (std::uint32_t l = 0; l < nl; ++l) off[l + 1] = off[l] + index.postings[l].size();
        ids.reserve(off[nl]);
        codes.reserve(off[nl] * m);
        for (const auto& list : index.postings)
            for (const auto& e : list) {
                ids.push_back(e.chunk_id);
                codes.insert(codes.end(), e.code.begin(), e.code.end());
            }
        if (devices.size() > 1)
            return from_host_sharded(nl, d, m, cent.data(), words.data(), off.data(), ids.data(), codes.data(),
                                     devices);
        return from_host(nl, d, m, cent.data(), words.data(), off.data(), ids.data(), codes.data(), devices.at(0));
    }
#endif

    Index(Index&&) noexcept = default;
    Index& operator=(Index&&) noexcept = default;

    prag_gpu_index* handle() const { return h_.get(); }
    // prag::store_index (annindex.hpp:335-359) of the resident index.
    void store(const std::string& pragix01_path) const { check(prag_gpu_index_store(h_.get(), pragix01_path.c_str())); }
    std::uint32_t nlist() const { return prag_gpu_index_nlist(h_.get()); }
    // Raw embeddings [n][d] by chunk id for exact rerank (annindex.hpp:307-312).
    void set_embeddings(const float* rows, std::uint64_t n) { check(prag_gpu_index_set_embeddings(h_.get(), rows, n)); }
    void set_embeddings(const std::vector<std::vector<float>>& e) {
        std::vector<float> flat;
        for (const auto& r : e) flat.insert(flat.end(), r.begin(), r.end());
        set_embeddings(flat.data(), e.size());
        attached_ = &e;
    }
    const void* attached() const { return attached_; }
    prag_gpu_index_desc describe() const {
        prag_gpu_index_desc d{};
        check(prag_gpu_index_describe(h_.get(), &d));
        return d;
    }

private:
    struct Free {
        void operator()(prag_gpu_index* p) const { prag_gpu_index_free(p); }
    };
    explicit Index(prag_gpu_index* h) : h_(h) {}
    std::unique_ptr<prag_gpu_index, Free> h_;
    const void* attached_ = nullptr;  // the embeddings object last given to set_embeddings
};

// Batch search; queries row-major nq x d (host or device pointer). Returns one
// SearchResult per query, exactly as nq calls of prag::search would.
// exact_rerank uses the embeddings attached with Index::set_embeddings
// (ConfigError "search: exact_rerank requires raw embeddings" otherwise).
inline std::vector<SearchResult> search_batch(const Index& index, const float* queries, std::uint32_t nq,
                                              SearchParams params, void* stream = nullptr) {
    const std::uint32_t k = params.k;
    std::vector<std::uint64_t> ids(std::size_t(nq) * (k ? k : 1));
    std::vector<float> dist(ids.size());
    std::vector<std::uint32_t> cnt(nq);
    std::vector<std::uint64_t> scanned(nq);
    auto fn = params.exact_rerank ? prag_gpu_search_rerank : prag_gpu_search;
    check(fn(index.handle(), queries, nq, params.nprobe, k, ids.data(), dist.data(), cnt.data(), scanned.data(),
             stream));
    std::vector<SearchResult> out(nq);
    for (std::uint32_t q = 0; q < nq; ++q) {
        out[q].scanned_vectors = scanned[q];
        out[q].scanned_lists = params.nprobe;  // annindex.hpp:284 counts empty lists too
        out[q].neighbors.resize(cnt[q]);
        for (std::uint32_t i = 0; i < cnt[q]; ++i)
            out[q].neighbors[i] = {ids[std::size_t(q) * k + i], dist[std::size_t(q) * k + i]};
    }
    return out;
}

// prag::search (annindex.hpp:262-315) for one query.
inline SearchResult search(const Index& index, const std::vector<float>& query, SearchParams params) {
    if (query.size() != index.describe().d) throw ConfigError("search: query dimension mismatch");
    return std::move(search_batch(index, query.data(), 1, params)[0]);
}

// prag::search(index, codebook, query, params, embeddings) (annindex.hpp:262-264):
// with exact_rerank the embeddings are attached to the device index (once per object).
inline SearchResult search(Index& index, const std::vector<float>& query, SearchParams params,
                           const std::vector<std::vector<float>>* embeddings) {
    if (params.exact_rerank && embeddings == nullptr)  // annindex.hpp:269-271
        throw ConfigError("search: exact_rerank requires raw embeddings");
    if (params.exact_rerank && index.attached() != embeddings) index.set_embeddings(*embeddings);
    return search(static_cast<const Index&>(index), query, params);
}

// perfmodel.hpp:92-117 fed with the GPU batch-latency curve: host queries in,
// host results out, wall clock per batch; median of `repeats` after `warmups`.
inline RetrievalPerfModel calibrate_retrieval(const Index& index, const float* queries, std::uint32_t nq,
                                              std::uint32_t k, const std::vector<std::uint32_t>& grid,
                                              int repeats = 5, int warmups = 2,
                                              std::vector<double>* latency_s = nullptr) {
    prag_gpu_perf_model m{};
    std::vector<double> lat(grid.size() + 1);
    check(prag_gpu_calibrate_retrieval(index.handle(), queries, nq, k, grid.data(), std::uint32_t(grid.size()),
                                       repeats, warmups, &m, lat.data()));
    if (latency_s) *latency_s = lat;
    return {m.slope_s, m.intercept_s, m.fit_residual_s, m.clamped != 0};
}

// perfmodel.hpp:148-157.
inline std::uint32_t select_nprobe(const RetrievalPerfModel& model, double budget_s, std::uint32_t nlist,
                                   double safety_margin = 0.10) {
    prag_gpu_perf_model m{model.slope_s, model.intercept_s, model.fit_residual_s, model.clamped ? 1 : 0, 0};
    return prag_gpu_select_nprobe(&m, budget_s, nlist, safety_margin);
}

#ifdef PRAG_GPU_HAVE_REFERENCE
// Drop-in for prag::train_index (annindex.hpp:164-241): the identical
// {IvfIndex, PqCodebook} (same sample, seeds, Lloyd iterations, lists in
// vector order, codebooks, codes), computed on `device`.
inline std::pair<::prag::IvfIndex, ::prag::PqCodebook> train_index(
    const std::vector<std::vector<float>>& embeddings, ::prag::TrainParams params, int device = 0) {
    const std::uint64_t n = embeddings.size();
    const std::uint32_t d = n ? static_cast<std::uint32_t>(embeddings[0].size()) : 0;
    std::vector<float> flat(n * d);
    for (std::uint64_t i = 0; i < n; ++i) {
        if (embeddings[i].size() != d) throw ConfigError("train_index: ragged embedding set");
        std::copy(embeddings[i].begin(), embeddings[i].end(), flat.begin() + i * d);
    }
    const std::uint32_t nsq = params.n_subquantizers ? params.n_subquantizers : std::max(1u, d / 4);
    const std::uint32_t sub = nsq && d % nsq == 0 ? d / nsq : 1;
    prag_gpu_train_params p{params.nlist, params.n_subquantizers, params.seed, params.kmeans_iterations, 0,
                            static_cast<std::uint64_t>(params.train_sample_cap)};
    std::vector<float> cent(std::size_t(params.nlist) * d + 1), words(std::size_t(nsq) * 256 * sub + 1);
    std::vector<std::uint64_t> off(std::size_t(params.nlist) + 1), ids(n + 1);
    std::vector<std::uint8_t> codes(n * nsq + 1);
    check(prag_gpu_train_index(n ? flat.data() : nullptr, n, d, &p, device, cent.data(), words.data(), off.data(),
                               ids.data(), codes.data()));
    ::prag::IvfIndex index;
    index.nlist = params.nlist;
    index.d = d;
    index.centroids.resize(params.nlist);
    index.postings.resize(params.nlist);
    for (std::uint32_t l = 0; l < params.nlist; ++l) {
        index.centroids[l].assign(cent.begin() + std::size_t(l) * d, cent.begin() + std::size_t(l + 1) * d);
        auto& list = index.postings[l];
        list.resize(off[l + 1] - off[l]);
        for (std::uint64_t e = off[l]; e < off[l + 1]; ++e) {
            auto& pe = list[e - off[l]];
            pe.chunk_id = ids[e];
            pe.code.assign(codes.begin() + e * nsq, codes.begin() + (e + 1) * nsq);
        }
    }
    ::prag::PqCodebook cb;
    cb.n_subquantizers = nsq;
    cb.sub_dim = sub;
    cb.codewords.assign(nsq, std::vector<std::vector<float>>(256, std::vector<float>(sub)));
    for (std::uint32_t s = 0; s < nsq; ++s)
        for (std::uint32_t c = 0; c < 256; ++c)
            std::copy(words.begin() + (std::size_t(s) * 256 + c) * sub,
                      words.begin() + (std::size_t(s) * 256 + c + 1) * sub, cb.codewords[s][c].begin());
    return {std::move(index), std::move(cb)};
}
#endif

#ifdef PRAG_GPU_HAVE_REFERENCE
// Drop-in for prag::LocalRetriever (pipeline.hpp:213-249): same constructor
// arguments, same nprobe directive handling (:224-226), same record
// resolution (:232-235). The query embedding (:227) and the search run on the
// B200: prag_gpu_embed reproduces ChunkEmbedder::embed bit for bit from
// token vectors computed on the host for the database's vocabulary.
// Re-entrant for concurrent callers (service.hpp:303, :338): each search
// uses its own stream-ordered workspace inside the library; the embedder's
// staging buffers are guarded by a mutex here.
class GpuRetriever : public ::prag::Retriever {
public:
    GpuRetriever(const ::prag::Database& db, const ::prag::IvfIndex& index, const ::prag::PqCodebook& codebook,
                 std::uint64_t embed_seed, ::prag::RetrievalPerfModel perf = {}, double safety_margin = 0.10,
                 int device = 0)
        : db_(&db), gpu_(Index::from_reference(index, codebook, device)), nlist_(index.nlist),
          embedder_(make_embedder(db, embed_seed, device)), perf_(perf), safety_margin_(safety_margin) {}

    // The index list-sharded over several GPUs (devices[0] embeds and merges).
    GpuRetriever(const ::prag::Database& db, const ::prag::IvfIndex& index, const ::prag::PqCodebook& codebook,
                 std::uint64_t embed_seed, ::prag::RetrievalPerfModel perf, double safety_margin,
                 const std::vector<int>& devices)
        : db_(&db), gpu_(Index::from_reference(index, codebook, devices)), nlist_(index.nlist),
          embedder_(make_embedder(db, embed_seed, devices.at(0))), perf_(perf), safety_margin_(safety_margin) {}

    GpuRetriever(const ::prag::Database& db, Index gpu_index, std::uint64_t embed_seed,
                 ::prag::RetrievalPerfModel perf = {}, double safety_margin = 0.10)
        : db_(&db), gpu_(std::move(gpu_index)), nlist_(gpu_.nlist()),
          embedder_(make_embedder(db, embed_seed, gpu_.describe().device)), perf_(perf),
          safety_margin_(safety_margin) {}

    // pipeline.hpp:224-226: the directive's nprobe (auto: from the perf model).
    std::uint32_t resolve_nprobe(const ::prag::NprobeDirective& directive) const {
        return directive.auto_mode ? ::prag::select_nprobe(perf_, directive.budget_s, nlist_, safety_margin_)
                                   : std::min(directive.nprobe, nlist_);
    }

    // Several queries that share k and nprobe in one embed + one batched
    // search (the serving path: GpuRetrievalService coalesces concurrent
    // requests through this). Outcome i is what retrieve(*queries[i], ...)
    // returns.
    std::vector<::prag::RetrievalOutcome> retrieve_batch(const std::vector<const ::prag::TokenChunk*>& queries,
                                                         std::uint32_t k, std::uint32_t nprobe) {
        ::prag::Stopwatch clock;
        const std::uint32_t nq = static_cast<std::uint32_t>(queries.size());
        std::vector<::prag::RetrievalOutcome> out(nq);
        if (nq == 0) return out;
        std::vector<float> emb(std::size_t(nq) * db_->d);
        const std::size_t m = queries[0]->size();
        bool same_len = true;
        for (const auto* q : queries) same_len = same_len && q->size() == m;
        {
            std::lock_guard<std::mutex> lk(embed_mu_);
            if (same_len) {
                std::vector<::prag::TokenId> toks;
                toks.reserve(nq * m);
                for (const auto* q : queries) toks.insert(toks.end(), q->begin(), q->end());
                check(prag_gpu_embed(embedder_.get(), toks.data(), nq, std::uint32_t(m), emb.data(), nullptr));
            } else {
                for (std::uint32_t i = 0; i < nq; ++i)
                    check(prag_gpu_embed(embedder_.get(), queries[i]->data(), 1, std::uint32_t(queries[i]->size()),
                                         emb.data() + std::size_t(i) * db_->d, nullptr));
            }
        }
        auto found = search_batch(gpu_, emb.data(), nq, SearchParams{nprobe, k, false});
        const double t = clock.elapsed_s();
        for (std::uint32_t i = 0; i < nq; ++i) {
            out[i].nprobe_used = nprobe;
            for (const auto& hit : found[i].neighbors) {
                const auto& rec = db_->records[hit.chunk_id];
                out[i].neighbors.push_back({rec.tokens, rec.continuation, hit.distance});
            }
            out[i].server_latency_s = t;
        }
        return out;
    }

    ::prag::RetrievalOutcome retrieve(const ::prag::TokenChunk& query_tokens, std::uint32_t k,
                                      ::prag::NprobeDirective directive) override {
        ::prag::Stopwatch clock;
        const std::uint32_t nprobe = resolve_nprobe(directive);
        std::vector<float> query(db_->d);
        {
            std::lock_guard<std::mutex> lk(embed_mu_);
            check(prag_gpu_embed(embedder_.get(), query_tokens.data(), 1, std::uint32_t(query_tokens.size()),
                                 query.data(), nullptr));
        }
        auto found = search_batch(gpu_, query.data(), 1, SearchParams{nprobe, k, false})[0];
        ::prag::RetrievalOutcome outcome;
        outcome.nprobe_used = nprobe;
        for (const auto& hit : found.neighbors) {
            const auto& rec = db_->records[hit.chunk_id];
            outcome.neighbors.push_back({rec.tokens, rec.continuation, hit.distance});
        }
        outcome.server_latency_s = clock.elapsed_s();
        return outcome;
    }

    std::uint32_t nlist() const override { return nlist_; }
    const Index& index() const { return gpu_; }

    // Recalibrates the retrieval model on this GPU's batch-1 latency curve
    // (the model is per batch size) and adopts it.
    ::prag::RetrievalPerfModel recalibrate(const std::vector<std::vector<float>>& queries,
                                           const std::vector<std::uint32_t>& grid, std::uint32_t k = 2,
                                           int repeats = 5) {
        std::vector<float> flat;
        for (const auto& q : queries) flat.insert(flat.end(), q.begin(), q.end());
        auto m = calibrate_retrieval(gpu_, flat.data(), std::uint32_t(queries.size()), k, grid, repeats, 2);
        perf_ = ::prag::RetrievalPerfModel{m.slope_s, m.intercept_s, m.fit_residual_s, m.clamped};
        return perf_;
    }

private:
    struct FreeEmbedder {
        void operator()(prag_gpu_embedder* e) const { prag_gpu_embedder_free(e); }
    };
    using EmbedderPtr = std::unique_ptr<prag_gpu_embedder, FreeEmbedder>;

    // Token vectors for every id the database uses (at least the byte
    // vocabulary, kByteVocabSize, common.hpp:21).
    static EmbedderPtr make_embedder(const ::prag::Database& db, std::uint64_t seed, int device) {
        std::uint32_t vocab = ::prag::kByteVocabSize;
        for (const auto& rec : db.records) {
            for (auto t : rec.tokens) vocab = std::max<std::uint32_t>(vocab, t + 1);
            for (auto t : rec.continuation) vocab = std::max<std::uint32_t>(vocab, t + 1);
        }
        prag_gpu_embedder* e = nullptr;
        check(prag_gpu_embedder_create(db.d, seed, vocab, device, &e));
        return EmbedderPtr(e);
    }

    const ::prag::Database* db_;
    Index gpu_;
    std::uint32_t nlist_;
    EmbedderPtr embedder_;
    std::mutex embed_mu_;
    ::prag::RetrievalPerfModel perf_;
    double safety_margin_;
};
#endif

}  // namespace gpu
}  // namespace prag
