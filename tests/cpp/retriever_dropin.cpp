// retriever_dropin.cpp -- TEST: the C++ drop-in boundary on a B200.
//
// Compiled by oracle/Makefile against the UNMODIFIED reference headers
// (/root/reference/proj/include, the integrator's tree) plus include/prag_gpu.hpp,
// linked with libprag_gpu.so, into oracle/_ref/retriever_dropin (git-ignored,
// travels to the GPU box). Run by tests/test_gpu_dropin.py.
//
// It swaps prag::LocalRetriever (pipeline.hpp:213-249) for
// prag::gpu::GpuRetriever on the same Database / IvfIndex / PqCodebook objects
// and requires the RetrievalOutcome of every retrieve() to be identical
// (Neighbor::operator== compares tokens, continuation and the float
// distance bit-for-bit), then replays reference test_annindex.cpp KATs
// through prag::gpu::search.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "prag_gpu.hpp"

using namespace prag;

namespace {

int g_fail = 0;

void report(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++g_fail;
}

std::vector<TokenId> random_tokens(SplitMix64& rng, std::size_t n) {
    std::vector<TokenId> t(n);
    for (auto& x : t) x = 1 + static_cast<TokenId>(rng.next_below(256));
    return t;
}

struct Fixture {
    Database db;
    IvfIndex index;
    PqCodebook codebook;
    Fixture(int docs, std::uint32_t d, std::uint32_t nlist, std::uint32_t nsq) {
        SplitMix64 rng(101);
        Corpus corpus;
        for (int i = 0; i < docs; ++i) corpus.documents.push_back(random_tokens(rng, 6400));
        db = build_database(corpus, 64, d, 7);
        TrainParams p;
        p.nlist = nlist;
        p.n_subquantizers = nsq;
        std::tie(index, codebook) = train_index(db.embeddings, p);
    }
};

bool same_outcome(const RetrievalOutcome& a, const RetrievalOutcome& b) {
    return a.nprobe_used == b.nprobe_used && a.neighbors == b.neighbors;
}

// devices: {} = one GPU; several entries = the index list-sharded over them
// (repeated ordinals put several shards on one GPU)
void dropin_parity(const Fixture& fx, const std::string& tag, const std::vector<int>& devices = {}) {
    RetrievalPerfModel perf{2e-5, 1e-4, 0.0, false};
    LocalRetriever local(fx.db, fx.index, fx.codebook, 7, perf);
    gpu::GpuRetriever gpu_r = devices.empty() ? gpu::GpuRetriever(fx.db, fx.index, fx.codebook, 7, perf)
                                              : gpu::GpuRetriever(fx.db, fx.index, fx.codebook, 7, perf, 0.10, devices);
    if (!devices.empty())
        report(gpu_r.index().describe().shard_world == int(devices.size()),
               tag + ": the retriever's index spans " + std::to_string(devices.size()) + " shards");
    report(gpu_r.nlist() == local.nlist(), tag + ": nlist()");
    SplitMix64 rng(202);
    int bad = 0, total = 0;
    for (int q = 0; q < 64; ++q) {
        // query = a stored chunk with a few tokens replaced (a stale window)
        TokenChunk chunk = fx.db.records[rng.next_below(fx.db.size())].tokens;
        for (int r = 0; r < 8; ++r) chunk[rng.next_below(chunk.size())] = 1 + TokenId(rng.next_below(256));
        for (std::uint32_t k : {1u, 2u, 10u}) {
            for (std::uint32_t np : {1u, 4u, 16u, fx.index.nlist, fx.index.nlist + 5}) {
                auto a = local.retrieve(chunk, k, NprobeDirective::fixed(np));
                auto b = gpu_r.retrieve(chunk, k, NprobeDirective::fixed(np));
                ++total;
                if (!same_outcome(a, b)) ++bad;
            }
            for (double budget : {0.0, 1e-4, 3e-4, 1e-2}) {
                auto a = local.retrieve(chunk, k, NprobeDirective::automatic(budget));
                auto b = gpu_r.retrieve(chunk, k, NprobeDirective::automatic(budget));
                ++total;
                if (!same_outcome(a, b)) ++bad;
            }
        }
    }
    report(bad == 0, tag + ": GpuRetriever == LocalRetriever on " + std::to_string(total) +
                         " retrievals (" + std::to_string(bad) + " differ)");

    // concurrent callers share one retriever (service.hpp:303, :338, :354)
    std::vector<std::thread> th;
    std::vector<int> errs(4, 0);
    for (int t = 0; t < 4; ++t)
        th.emplace_back([&, t] {
            SplitMix64 r2(300 + t);
            for (int i = 0; i < 16; ++i) {
                const auto& chunk = fx.db.records[r2.next_below(fx.db.size())].tokens;
                auto a = local.retrieve(chunk, 2, NprobeDirective::fixed(8));
                auto b = gpu_r.retrieve(chunk, 2, NprobeDirective::fixed(8));
                if (!same_outcome(a, b)) ++errs[t];
            }
        });
    for (auto& t : th) t.join();
    report(errs[0] + errs[1] + errs[2] + errs[3] == 0, tag + ": 4 concurrent threads on one GpuRetriever");

    // raw search: batch == per-query reference search(), incl. scanned_vectors
    std::vector<float> flat;
    std::vector<std::vector<float>> qs;
    SplitMix64 r3(13);
    for (int q = 0; q < 32; ++q) {
        auto v = fx.db.embeddings[r3.next_below(fx.db.size())];
        for (auto& x : v) x += 0.05f * static_cast<float>(r3.next_gaussian());
        qs.push_back(v);
        flat.insert(flat.end(), v.begin(), v.end());
    }
    bad = 0;
    for (std::uint32_t np : {1u, 8u, fx.index.nlist}) {
        auto got = gpu::search_batch(gpu_r.index(), flat.data(), 32, {np, 10, false});
        for (int q = 0; q < 32; ++q) {
            auto ref = search(fx.index, fx.codebook, qs[q], {np, 10, false});
            bool ok = ref.neighbors.size() == got[q].neighbors.size() &&
                      ref.scanned_vectors == got[q].scanned_vectors && ref.scanned_lists == got[q].scanned_lists;
            for (std::size_t i = 0; ok && i < ref.neighbors.size(); ++i)
                ok = ref.neighbors[i].chunk_id == got[q].neighbors[i].chunk_id &&
                     ref.neighbors[i].distance == got[q].neighbors[i].distance;
            if (!ok) ++bad;
        }
    }
    report(bad == 0, tag + ": search_batch == prag::search (ids, distances, scanned_vectors)");
}

void kats() {
    // test_annindex.cpp:176-192: parameter validation surfaces prag::ConfigError
    std::vector<std::vector<float>> vecs;
    SplitMix64 rng(5);
    for (int i = 0; i < 600; ++i) {
        std::vector<float> v(16);
        for (auto& x : v) x = static_cast<float>(rng.next_gaussian());
        vecs.push_back(v);
    }
    TrainParams p;
    p.nlist = 8;
    auto [index, cb] = train_index(vecs, p);
    auto g = gpu::Index::from_reference(index, cb);
    auto throws_config = [&](gpu::SearchParams sp) {
        try {
            gpu::search(g, vecs[0], sp);
        } catch (const ConfigError&) {
            return true;
        }
        return false;
    };
    report(throws_config({0, 2, false}), "nprobe 0 -> ConfigError");
    report(throws_config({9, 2, false}), "nprobe > nlist -> ConfigError");
    report(throws_config({1, 0, false}), "k 0 -> ConfigError");
    report(throws_config({1, 2, true}), "rerank without embeddings -> ConfigError");
    // test_annindex.cpp:39-48: every vector finds itself first at full probe
    bool self = true;
    for (int i = 0; i < 600 && self; i += 37) {
        auto r = gpu::search(g, vecs[i], {8, 1, false});
        auto ref = search(index, cb, vecs[i], {8, 1, false});
        self = r.neighbors.size() == 1 && r.neighbors[0].chunk_id == ref.neighbors[0].chunk_id &&
               r.scanned_vectors == vecs.size();
    }
    report(self, "full probe: top-1 matches reference, scanned_vectors == n");
    // load_index on a missing file -> FormatError
    bool fe = false;
    try {
        gpu::Index::load("/nonexistent/idx.pragix");
    } catch (const FormatError&) {
        fe = true;
    }
    report(fe, "missing index file -> FormatError");
    // select_nprobe KATs (test_perfmodel.cpp:54-68) through the GPU model API
    gpu::RetrievalPerfModel m{0.001, 0.004, 0, false};
    report(gpu::select_nprobe(m, 0.02, 64, 0.0) == 16 && select_nprobe({0.001, 0.004, 0, false}, 0.02, 64, 0.0) == 16,
           "select_nprobe KAT (16)");
}

}  // namespace

int main() {
    if (prag_gpu_device_count() < 1) {
        std::printf("no CUDA device\n");
        return 2;
    }
    kats();
    {
        // prag::gpu::train_index == prag::train_index on the same embeddings
        SplitMix64 rng(77);
        Corpus corpus;
        for (int i = 0; i < 40; ++i) corpus.documents.push_back(random_tokens(rng, 6400));
        Database db = build_database(corpus, 64, 96, 7);
        TrainParams p;
        p.nlist = 24;
        p.n_subquantizers = 24;
        p.train_sample_cap = 2000;
        auto [ri, rc] = train_index(db.embeddings, p);
        auto [gi, gc] = gpu::train_index(db.embeddings, p);
        bool same = ri.nlist == gi.nlist && ri.d == gi.d && ri.centroids == gi.centroids &&
                    rc.n_subquantizers == gc.n_subquantizers && rc.sub_dim == gc.sub_dim &&
                    rc.codewords == gc.codewords && ri.postings.size() == gi.postings.size();
        for (std::size_t l = 0; same && l < ri.postings.size(); ++l) {
            same = ri.postings[l].size() == gi.postings[l].size();
            for (std::size_t e = 0; same && e < ri.postings[l].size(); ++e)
                same = ri.postings[l][e].chunk_id == gi.postings[l][e].chunk_id &&
                       ri.postings[l][e].code == gi.postings[l][e].code;
        }
        report(same, "gpu::train_index == prag::train_index (" + std::to_string(db.size()) + " chunks, d=96)");
    }
    {
        Fixture fx(60, 32, 32, 0);  // d=32, nsq=8 (reference defaults): generic scan path
        dropin_parity(fx, "d32/m8");
    }
    {
        Fixture fx(60, 384, 32, 32);  // d=384, m=32: lane-skewed fast path
        dropin_parity(fx, "d384/m32");
        // list-sharded GpuRetriever: 3 shards (each on GPU 0 here; on an
        // 8-GPU box pass {0, 1, 2, ...}) merged by the peer-memory kernel
        dropin_parity(fx, "d384/m32 sharded x3", {0, 0, 0});
    }
    {
        Fixture fx(60, 32, 32, 0);
        dropin_parity(fx, "d32/m8 sharded x2", {0, 0});
    }
    std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASS", g_fail);
    return g_fail ? 1 : 0;
}
