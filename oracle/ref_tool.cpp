// ref_tool.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Thin driver around the UNMODIFIED reference headers
// (/root/reference/proj/include/prag/annindex.hpp, perfmodel.hpp), compiled by
// oracle/Makefile with the reference's own CMake Release flags into
// oracle/_ref/ref_tool. It is used (a) to generate the golden fixtures in
// tests/golden/ with the reference's own train_index/store_index/search, and
// (b) as the CPU baseline / `bench.py --impl reference` arm, timing
// prag::search on indexes loaded with prag::load_index (as every reference
// tool does: perfmodel_main.cpp:49). No reference source is copied here.
//
// Commands:
//   train   <vectors.f32> <n> <d> <nlist> <nsq> <seed> <out.pragix> [iterations] [sample_cap]
//   search  <index> <queries.f32> <nq> <nprobe> <k> <out.bin>
//   bench   <index> <queries.f32> <nq> <nprobe> <k> <threads> <reps> <warmups> [max_seconds] [out.bin]
//           (out.bin: the last timed batch's results, for bench.py's parity check)
//   calibrate <index> <queries.f32> <nq> <k> <grid_csv> <repeats>
//   brute   <vectors.f32> <n> <d> <queries.f32> <nq> <k> <out.bin>
//   rerank  <index> <vectors.f32> <n> <queries.f32> <nq> <nprobe> <k> <out.bin>   (exact_rerank = true)
//   embed   <tokens.u32> <nchunks> <m> <d> <seed> <out.f32>   (prag::ChunkEmbedder::embed)
//   synth-search <cents.f32> <words.f32> <sizes.u64> <nlist> <d> <nsq> <seed> <queries.f32> <nq> <nprobe> <k> <out.bin>
//   synth-bench  <cents.f32> <words.f32> <sizes.u64> <nlist> <d> <nsq> <seed> <queries.f32> <nq> <nprobe> <k>
//                <threads> <reps> <warmups> <max_seconds>
//           (the device-built synthetic index, prag_gpu_index_synthetic, rebuilt as the reference's
//            IvfIndex/PqCodebook from the same list sizes and code formula; configs C/D)
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "prag/annindex.hpp"
#include "prag/perfmodel.hpp"
#include "prag/tokendb.hpp"

namespace {

std::vector<float> read_f32(const std::string& path, std::size_t count) {
    std::vector<float> v(count);
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::runtime_error("cannot open " + path);
    is.read(reinterpret_cast<char*>(v.data()), count * sizeof(float));
    if (!is) throw std::runtime_error("short read " + path);
    return v;
}

std::vector<std::vector<float>> rows(const std::vector<float>& flat, std::size_t n, std::size_t d) {
    std::vector<std::vector<float>> out(n, std::vector<float>(d));
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < d; ++j) out[i][j] = flat[i * d + j];
    return out;
}

// Result file: per query u32 count, u32 scanned_lists, u64 scanned_vectors,
// then k x (u64 id, f32 dist), unused slots zero.
void write_results(const std::string& path, const std::vector<prag::SearchResult>& res, std::uint32_t k) {
    std::ofstream os(path, std::ios::binary);
    for (const auto& r : res) {
        std::uint32_t count = static_cast<std::uint32_t>(r.neighbors.size());
        os.write(reinterpret_cast<const char*>(&count), 4);
        os.write(reinterpret_cast<const char*>(&r.scanned_lists), 4);
        os.write(reinterpret_cast<const char*>(&r.scanned_vectors), 8);
        for (std::uint32_t i = 0; i < k; ++i) {
            std::uint64_t id = i < count ? r.neighbors[i].chunk_id : 0;
            float dist = i < count ? r.neighbors[i].distance : 0.0f;
            os.write(reinterpret_cast<const char*>(&id), 8);
            os.write(reinterpret_cast<const char*>(&dist), 4);
        }
    }
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

std::vector<std::uint64_t> read_u64(const std::string& path, std::size_t count) {
    std::vector<std::uint64_t> v(count);
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::runtime_error("cannot open " + path);
    is.read(reinterpret_cast<char*>(v.data()), count * 8);
    if (!is) throw std::runtime_error("short read " + path);
    return v;
}

// splitmix64 finaliser (common.hpp:37-52's mixing steps), as the device's
// synthetic code formula uses it (include/prag_gpu.h, prag_gpu_index_synthetic)
std::uint64_t fin64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void synth_index(const std::vector<float>& cents, const std::vector<float>& words, const std::vector<std::uint64_t>& sizes,
                 std::uint32_t nlist, std::uint32_t d, std::uint32_t nsq, std::uint64_t seed, prag::IvfIndex& index,
                 prag::PqCodebook& codebook) {
    const std::uint32_t sub = d / nsq;
    index.nlist = nlist;
    index.d = d;
    index.centroids.assign(nlist, std::vector<float>(d));
    for (std::uint32_t c = 0; c < nlist; ++c)
        for (std::uint32_t j = 0; j < d; ++j) index.centroids[c][j] = cents[std::size_t(c) * d + j];
    codebook.n_subquantizers = nsq;
    codebook.sub_dim = sub;
    codebook.codewords.assign(nsq, std::vector<std::vector<float>>(256, std::vector<float>(sub)));
    for (std::uint32_t s = 0; s < nsq; ++s)
        for (std::uint32_t c = 0; c < 256; ++c)
            for (std::uint32_t j = 0; j < sub; ++j)
                codebook.codewords[s][c][j] = words[(std::size_t(s) * 256 + c) * sub + j];
    index.postings.assign(nlist, {});
    std::uint64_t g = 0;
    for (std::uint32_t l = 0; l < nlist; ++l) {
        auto& pl = index.postings[l];
        pl.resize(sizes[l]);
        for (auto& e : pl) {
            e.chunk_id = g;
            e.code.resize(nsq);
            for (std::uint32_t i = 0; i < nsq / 8; ++i) {
                const std::uint64_t w = fin64(seed + 8 * g + i + 0x9e3779b97f4a7c15ULL);
                for (int b = 0; b < 8; ++b) e.code[8 * i + b] = std::uint8_t(w >> (8 * b));
            }
            ++g;
        }
    }
}

// nq queries by `threads` std::threads pulling query indices from an atomic
// counter (prag::search is re-entrant); p50 over `reps` batches
void bench_loop(const prag::IvfIndex& index, const prag::PqCodebook& codebook, const std::vector<std::vector<float>>& qs,
                std::uint32_t nprobe, std::uint32_t k, int threads, int reps, int warm, double max_s,
                const std::string& out_path, double t_load) {
    const std::size_t nq = qs.size();
    std::vector<prag::SearchResult> last(nq);
    if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
    std::vector<double> times;
    std::uint64_t scanned = 0;
    double t_begin = now_s();
    for (int r = 0; r < warm + reps; ++r) {
        std::atomic<std::size_t> next{0};
        std::atomic<std::uint64_t> sc{0};
        double t0 = now_s();
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&] {
                for (;;) {
                    std::size_t q = next.fetch_add(1);
                    if (q >= nq) break;
                    auto res = prag::search(index, codebook, qs[q], {nprobe, k, false});
                    sc += res.scanned_vectors;
                    last[q] = std::move(res);
                }
            });
        }
        for (auto& th : pool) th.join();
        double dt = now_s() - t0;
        if (r >= warm) times.push_back(dt);
        scanned = sc.load();
        if (r >= warm && now_s() - t_begin > max_s) break;
    }
    if (!out_path.empty()) write_results(out_path, last, k);
    std::vector<double> sorted = times;
    std::sort(sorted.begin(), sorted.end());
    double p50 = sorted[sorted.size() / 2];
    std::printf("{\"nq\": %zu, \"nprobe\": %u, \"k\": %u, \"threads\": %d, \"reps\": %zu, "
                "\"p50_s\": %.9g, \"best_s\": %.9g, \"qps\": %.6g, \"scanned_vectors\": %llu, "
                "\"load_s\": %.4g}\n",
                nq, nprobe, k, threads, times.size(), p50, sorted.front(), nq / p50,
                static_cast<unsigned long long>(scanned), t_load);
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: ref_tool train|search|bench|calibrate|brute ...\n";
        return 2;
    }
    std::string cmd = argv[1];
    try {
        if (cmd == "train" && argc >= 9 && argc <= 11) {
            std::size_t n = std::stoull(argv[3]);
            std::uint32_t d = std::stoul(argv[4]);
            prag::TrainParams params;
            params.nlist = std::stoul(argv[5]);
            params.n_subquantizers = std::stoul(argv[6]);
            params.seed = std::stoull(argv[7]);
            if (argc >= 10) params.kmeans_iterations = std::stoi(argv[9]);
            if (argc >= 11) params.train_sample_cap = std::stoull(argv[10]);
            auto vecs = rows(read_f32(argv[2], n * d), n, d);
            auto [index, codebook] = prag::train_index(vecs, params);
            prag::store_index(index, codebook, argv[8]);
            return 0;
        }
        if (cmd == "embed" && argc == 8) {
            const std::size_t nch = std::stoull(argv[3]), m = std::stoull(argv[4]);
            const std::uint32_t d = std::stoul(argv[5]);
            const std::uint64_t seed = std::stoull(argv[6]);
            std::vector<std::uint32_t> tok(nch * m);
            {
                std::ifstream is(argv[2], std::ios::binary);
                is.read(reinterpret_cast<char*>(tok.data()), tok.size() * 4);
                if (!is) throw std::runtime_error("short read tokens");
            }
            prag::ChunkEmbedder emb(d, seed);
            std::ofstream os(argv[7], std::ios::binary);
            for (std::size_t c = 0; c < nch; ++c) {
                prag::TokenChunk chunk(tok.begin() + c * m, tok.begin() + (c + 1) * m);
                const auto v = emb.embed(chunk);
                os.write(reinterpret_cast<const char*>(v.data()), v.size() * 4);
            }
            return 0;
        }
        if (cmd == "search" && argc == 8) {
            auto [index, codebook] = prag::load_index(argv[2]);
            std::size_t nq = std::stoull(argv[4]);
            std::uint32_t nprobe = std::stoul(argv[5]), k = std::stoul(argv[6]);
            auto qs = rows(read_f32(argv[3], nq * index.d), nq, index.d);
            std::vector<prag::SearchResult> res;
            for (const auto& q : qs) res.push_back(prag::search(index, codebook, q, {nprobe, k, false}));
            write_results(argv[7], res, k);
            return 0;
        }
        if (cmd == "rerank" && argc == 10) {  // search with exact_rerank (annindex.hpp:307-312)
            auto [index, codebook] = prag::load_index(argv[2]);
            std::size_t n = std::stoull(argv[4]);
            auto vecs = rows(read_f32(argv[3], n * index.d), n, index.d);
            std::size_t nq = std::stoull(argv[6]);
            std::uint32_t nprobe = std::stoul(argv[7]), k = std::stoul(argv[8]);
            auto qs = rows(read_f32(argv[5], nq * index.d), nq, index.d);
            std::vector<prag::SearchResult> res;
            for (const auto& q : qs) res.push_back(prag::search(index, codebook, q, {nprobe, k, true}, &vecs));
            write_results(argv[9], res, k);
            return 0;
        }
        if (cmd == "brute" && argc == 9) {
            std::size_t n = std::stoull(argv[3]);
            std::uint32_t d = std::stoul(argv[4]);
            std::size_t nq = std::stoull(argv[6]);
            std::uint32_t k = std::stoul(argv[7]);
            auto vecs = rows(read_f32(argv[2], n * d), n, d);
            auto qs = rows(read_f32(argv[5], nq * d), nq, d);
            std::vector<prag::SearchResult> res;
            for (const auto& q : qs) res.push_back(prag::brute_force_search(vecs, q, k));
            write_results(argv[8], res, k);
            return 0;
        }
        if (cmd == "bench" && argc >= 10 && argc <= 12) {
            double t_load0 = now_s();
            auto [index, codebook] = prag::load_index(argv[2]);
            double t_load = now_s() - t_load0;
            std::size_t nq = std::stoull(argv[4]);
            auto qs = rows(read_f32(argv[3], nq * index.d), nq, index.d);
            bench_loop(index, codebook, qs, std::stoul(argv[5]), std::stoul(argv[6]), std::stoi(argv[7]),
                       std::stoi(argv[8]), std::stoi(argv[9]), argc >= 11 ? std::stod(argv[10]) : 1e30,
                       argc == 12 ? argv[11] : "", t_load);
            return 0;
        }
        if ((cmd == "synth-bench" && argc == 17) || (cmd == "synth-search" && argc == 14)) {
            // the device-built synthetic index (prag_gpu_index_synthetic) as the
            // reference's own IvfIndex: list sizes from the GPU handle, entry g
            // (global, list-major) = chunk id g, code bytes from the formula
            const std::uint32_t nlist = std::stoul(argv[5]), d = std::stoul(argv[6]), nsq = std::stoul(argv[7]);
            const std::uint64_t seed = std::stoull(argv[8]);
            double t0 = now_s();
            prag::IvfIndex index;
            prag::PqCodebook codebook;
            synth_index(read_f32(argv[2], std::size_t(nlist) * d), read_f32(argv[3], std::size_t(d) * 256),
                        read_u64(argv[4], nlist), nlist, d, nsq, seed, index, codebook);
            double t_build = now_s() - t0;
            std::size_t nq = std::stoull(argv[10]);
            auto qs = rows(read_f32(argv[9], nq * d), nq, d);
            const std::uint32_t nprobe = std::stoul(argv[11]), k = std::stoul(argv[12]);
            if (cmd == "synth-search") {
                std::vector<prag::SearchResult> res;
                for (const auto& q : qs) res.push_back(prag::search(index, codebook, q, {nprobe, k, false}));
                write_results(argv[13], res, k);
                return 0;
            }
            bench_loop(index, codebook, qs, nprobe, k, std::stoi(argv[13]), std::stoi(argv[14]), std::stoi(argv[15]),
                       std::stod(argv[16]), "", t_build);
            return 0;
        }
        if (cmd == "calibrate" && argc == 8) {
            // perfmodel_main.cpp:57-70 protocol: per-query seconds, sequential.
            auto [index, codebook] = prag::load_index(argv[2]);
            std::size_t nq = std::stoull(argv[4]);
            std::uint32_t k = std::stoul(argv[5]);
            int repeats = std::stoi(argv[7]);
            auto qs = rows(read_f32(argv[3], nq * index.d), nq, index.d);
            std::vector<std::uint32_t> grid;
            std::stringstream ss(argv[6]);
            std::string item;
            while (std::getline(ss, item, ',')) grid.push_back(std::stoul(item));
            auto measure = [&](std::uint32_t nprobe) {
                prag::Stopwatch clock;
                for (const auto& q : qs) prag::search(index, codebook, q, {nprobe, k, false});
                return clock.elapsed_s() / qs.size();
            };
            auto model = prag::calibrate_retrieval(measure, grid, repeats);
            std::printf("{\"slope_s\": %.9g, \"intercept_s\": %.9g, \"fit_residual_s\": %.9g, \"clamped\": %s}\n",
                        model.slope_s, model.intercept_s, model.fit_residual_s,
                        model.clamped ? "true" : "false");
            return 0;
        }
    } catch (const prag::ConfigError& e) {
        std::cerr << "ConfigError: " << e.what() << "\n";
        return 3;
    } catch (const prag::FormatError& e) {
        std::cerr << "FormatError: " << e.what() << "\n";
        return 4;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    std::cerr << "bad arguments\n";
    return 2;
}
