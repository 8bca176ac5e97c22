// service_dropin.cpp -- TEST: the retrieval service (PRAGRPC1, SURVEY.md 8(f)
// row 4) served from the B200.
//
// Compiled by oracle/Makefile against the UNMODIFIED reference headers plus
// include/prag_gpu_service.hpp, linked with libprag_gpu.so, into
// oracle/_ref/service_dropin (run by tests/test_gpu_service.py).
//
// The reference prag::RetrievalService (service.hpp:243-362, CPU
// LocalRetriever behind one thread per connection) and
// prag::gpu::GpuRetrievalService run side by side on loopback over the same
// Database / IvfIndex / PqCodebook. Reference prag::RetrievalClient
// connections send both the same requests; every response must match
// (request id, nprobe_used, neighbours bit for bit), including under
// concurrent clients (where the GPU service batches), and malformed frames
// must get the same error frames. Then both are timed with C concurrent
// clients; one JSON line per setting goes to stdout.
//
// usage: service_dropin [docs=200] [clients=16] [requests_per_client=100]
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "prag_gpu_service.hpp"

using namespace prag;

namespace {

int g_fail = 0;

void report(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    std::fflush(stdout);
    if (!ok) ++g_fail;
}

bool same(const RetrievalResponse& a, const RetrievalResponse& b) {
    return a.request_id == b.request_id && a.nprobe_used == b.nprobe_used && a.neighbors == b.neighbors;
}

// One raw frame exchange on a fresh connection (for malformed input).
std::vector<std::uint8_t> raw_exchange(std::uint16_t port, const std::vector<std::uint8_t>& bytes) {
    int fd = ::socket(AF_INET, SOCK_STREAM, 0);
    sockaddr_in addr{};
    addr.sin_family = AF_INET;
    addr.sin_port = htons(port);
    ::inet_pton(AF_INET, "127.0.0.1", &addr.sin_addr);
    if (::connect(fd, reinterpret_cast<sockaddr*>(&addr), sizeof(addr)) != 0) return {};
    detail::write_all(fd, bytes.data(), bytes.size());
    std::vector<std::uint8_t> out;
    char magic[8];
    std::uint32_t n = 0;
    if (detail::read_exact(fd, magic, 8, 5000) == 0 && detail::read_exact(fd, &n, 4, 5000) == 0 && n < 4096) {
        out.resize(n);
        if (detail::read_exact(fd, out.data(), n, 5000) != 0) out.clear();
    }
    ::close(fd);
    return out;
}

std::vector<RetrievalRequest> make_requests(const Database& db, std::uint64_t seed, int n, std::uint32_t nlist) {
    SplitMix64 rng(seed);
    std::vector<RetrievalRequest> reqs;
    for (int i = 0; i < n; ++i) {
        RetrievalRequest r;
        r.request_id = seed * 100000 + i;
        r.query_tokens = db.records[rng.next_below(db.size())].tokens;
        for (int j = 0; j < 6; ++j) r.query_tokens[rng.next_below(r.query_tokens.size())] = 1 + TokenId(rng.next_below(255));
        r.k = 1 + std::uint32_t(rng.next_below(10));
        switch (i % 4) {
            case 0: r.directive = NprobeDirective::fixed(8); break;
            case 1: r.directive = NprobeDirective::fixed(1 + std::uint32_t(rng.next_below(nlist + 8))); break;
            case 2: r.directive = NprobeDirective::automatic(2e-4); break;
            default: r.directive = NprobeDirective::fixed(32); break;
        }
        reqs.push_back(r);
    }
    return reqs;
}

double run_load(std::uint16_t port, int clients, int per_client, std::uint32_t k, std::uint32_t nprobe,
                const Database& db) {
    std::vector<std::thread> th;
    Stopwatch clock;
    for (int c = 0; c < clients; ++c)
        th.emplace_back([&, c] {
            RetrievalClient client("127.0.0.1", port);
            SplitMix64 rng(1000 + c);
            for (int i = 0; i < per_client; ++i) {
                RetrievalRequest r;
                r.request_id = i;
                r.k = k;
                r.directive = NprobeDirective::fixed(nprobe);
                r.query_tokens = db.records[rng.next_below(db.size())].tokens;
                client.retrieve(r);
            }
        });
    for (auto& t : th) t.join();
    return clients * per_client / clock.elapsed_s();
}

}  // namespace

int main(int argc, char** argv) {
    if (prag_gpu_device_count() < 1) {
        std::printf("no CUDA device\n");
        return 2;
    }
    const int docs = argc > 1 ? std::atoi(argv[1]) : 200;
    const int clients = argc > 2 ? std::atoi(argv[2]) : 16;
    const int per_client = argc > 3 ? std::atoi(argv[3]) : 100;

    SplitMix64 rng(101);
    Corpus corpus;
    for (int i = 0; i < docs; ++i) {
        std::vector<TokenId> t(6400);
        for (auto& x : t) x = 1 + static_cast<TokenId>(rng.next_below(256));
        corpus.documents.push_back(std::move(t));
    }
    Stopwatch build;
    Database db = build_database(corpus, 64, 384, 7);
    TrainParams tp;
    tp.nlist = 256;
    tp.n_subquantizers = 32;
    // the reference train_index's exact result, computed on the GPU (test_gpu_train.py)
    auto [index, codebook] = gpu::train_index(db.embeddings, tp);
    std::printf("db: %zu chunks, d=384, nlist=256, m=32 (built in %.1f s)\n", db.size(), build.elapsed_s());

    RetrievalPerfModel perf{2e-6, 5e-5, 0.0, false};
    RetrievalService ref(db, index, codebook, 7, perf);
    gpu::GpuRetrievalService gsvc(db, index, codebook, 7, perf);
    const std::uint16_t pr = ref.start(), pg = gsvc.start();

    // 1. sequential parity
    {
        RetrievalClient a("127.0.0.1", pr), b("127.0.0.1", pg);
        const auto reqs = make_requests(db, 5, 120, index.nlist);
        int bad = 0;
        for (const auto& r : reqs)
            if (!same(a.retrieve(r).response, b.retrieve(r).response)) ++bad;
        report(bad == 0, "sequential: " + std::to_string(reqs.size()) + " requests, " + std::to_string(bad) +
                             " responses differ");
    }
    // 2. concurrent clients (the GPU service batches them); reference answers
    //    computed afterwards, one by one
    {
        const int C = 12;
        std::vector<std::vector<RetrievalRequest>> reqs(C);
        std::vector<std::vector<RetrievalResponse>> got(C);
        for (int c = 0; c < C; ++c) reqs[c] = make_requests(db, 50 + c, 40, index.nlist);
        std::vector<std::thread> th;
        for (int c = 0; c < C; ++c)
            th.emplace_back([&, c] {
                RetrievalClient b("127.0.0.1", pg);
                for (const auto& r : reqs[c]) got[c].push_back(b.retrieve(r).response);
            });
        for (auto& t : th) t.join();
        RetrievalClient a("127.0.0.1", pr);
        int bad = 0, total = 0;
        for (int c = 0; c < C; ++c)
            for (std::size_t i = 0; i < reqs[c].size(); ++i, ++total)
                if (!same(a.retrieve(reqs[c][i]).response, got[c][i])) ++bad;
        const auto st = gsvc.batch_stats();
        report(bad == 0, "concurrent: " + std::to_string(C) + " clients x 40 requests, " + std::to_string(bad) +
                             " differ (GPU batches: " + std::to_string(st.batches) + ", largest " +
                             std::to_string(st.max_batch_seen) + ")");
    }
    // 3. malformed frames get the same error frames (service.hpp:309-331)
    {
        std::vector<std::uint8_t> bad_magic = {'X', 'X', 'X', 'X', 'X', 'X', 'X', 'X', 1, 0, 0, 0, 1};
        std::vector<std::uint8_t> bad_ver = {'P', 'R', 'A', 'G', 'R', 'P', 'C', '9', 1, 0, 0, 0, 1};
        std::vector<std::uint8_t> bad_type = {'P', 'R', 'A', 'G', 'R', 'P', 'C', '1', 1, 0, 0, 0, 0x42};
        std::vector<std::uint8_t> bad_len = {'P', 'R', 'A', 'G', 'R', 'P', 'C', '1', 0, 0, 0, 0};
        std::vector<std::uint8_t> bad_payload = {'P', 'R', 'A', 'G', 'R', 'P', 'C', '1', 3, 0, 0, 0, 1, 9, 9};
        int i = 0;
        for (const auto& f : {bad_magic, bad_ver, bad_type, bad_len, bad_payload}) {
            const auto x = raw_exchange(pr, f), y = raw_exchange(pg, f);
            report(!x.empty() && x == y, "error frame " + std::to_string(i++) + " identical (" +
                                             std::to_string(x.size()) + " bytes)");
        }
    }
    // 4. throughput: C clients, fixed k and nprobe (one untimed warm-up pass
    //    per service first: workspace and staging buffers reach their size)
    run_load(pr, clients, 8, 2, 32, db);
    run_load(pg, clients, 8, 2, 32, db);
    for (std::uint32_t nprobe : {8u, 32u, 128u}) {
        const double r_ref = run_load(pr, clients, per_client, 2, nprobe, db);
        const double r_gpu = run_load(pg, clients, per_client, 2, nprobe, db);
        std::printf("{\"bench\": \"service\", \"clients\": %d, \"requests_per_client\": %d, \"k\": 2, "
                    "\"nprobe\": %u, \"chunks\": %zu, \"reference_req_per_s\": %.1f, \"gpu_req_per_s\": %.1f}\n",
                    clients, per_client, nprobe, db.size(), r_ref, r_gpu);
    }
    const auto st = gsvc.batch_stats();
    std::printf("gpu batches: %llu requests in %llu batches (largest %llu)\n", (unsigned long long)st.requests,
                (unsigned long long)st.batches, (unsigned long long)st.max_batch_seen);
    ref.stop();
    gsvc.stop();
    std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASS", g_fail);
    return g_fail ? 1 : 0;
}
