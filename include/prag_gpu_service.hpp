// prag_gpu_service.hpp -- the reference's retrieval service (PRAGRPC1 over
// TCP, /root/reference/proj/include/prag/service.hpp:24-362) served from the
// B200, SURVEY.md 8(f) row 4.
//
// The wire format is the reference's own: frames are read and written with
// its encode_*/decode_* functions and detail::read_exact / send_frame
// (service.hpp:75-236), so the reference RetrievalClient and
// NetworkRetriever (:366-470) talk to this service unchanged, and error
// frames carry the same codes and texts (:309-345).
//
// What differs is the compute behind it. The reference gives every
// connection a thread that calls LocalRetriever::retrieve (CPU search,
// :338). Here connection threads only parse and answer frames; their
// requests go to one dispatcher thread that coalesces whatever is pending
// and shares (k, nprobe) into a single batched embed + search on the GPU
// (GpuRetriever::retrieve_batch), up to max_batch queries per launch. Under
// concurrency the GPU then sees batches instead of single queries.
//
// Header-only; needs the reference headers on the include path (like
// GpuRetriever) and libprag_gpu.so at link time.
#pragma once

#include <prag/service.hpp>

#include <condition_variable>
#include <deque>
#include <future>
#include <map>

#include "prag_gpu.hpp"

#ifndef PRAG_GPU_HAVE_REFERENCE
#error "prag_gpu_service.hpp needs the reference headers (prag/pipeline.hpp) on the include path"
#endif

namespace prag {
namespace gpu {

// A Retriever whose retrieve() calls are coalesced across threads into
// GpuRetriever::retrieve_batch calls. Requests are served in arrival order
// of their batch's first member; a batch takes every pending request with
// the same (k, nprobe), at most max_batch of them.
class BatchingRetriever : public ::prag::Retriever {
public:
    explicit BatchingRetriever(GpuRetriever& gpu, std::uint32_t max_batch = 64)
        : gpu_(&gpu), max_batch_(std::max<std::uint32_t>(1, max_batch)), worker_([this] { run(); }) {}

    ~BatchingRetriever() override {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        worker_.join();
    }

    BatchingRetriever(const BatchingRetriever&) = delete;
    BatchingRetriever& operator=(const BatchingRetriever&) = delete;

    ::prag::RetrievalOutcome retrieve(const ::prag::TokenChunk& query_tokens, std::uint32_t k,
                                      ::prag::NprobeDirective directive) override {
        Pending p{&query_tokens, k, gpu_->resolve_nprobe(directive), {}};
        auto fut = p.result.get_future();
        {
            std::lock_guard<std::mutex> lk(mu_);
            queue_.push_back(std::move(p));
        }
        cv_.notify_one();
        return fut.get();  // rethrows the batch's exception, if any
    }

    std::uint32_t nlist() const override { return gpu_->nlist(); }

    struct Stats {
        std::uint64_t requests = 0, batches = 0, max_batch_seen = 0;
    };
    Stats stats() const {
        std::lock_guard<std::mutex> lk(mu_);
        return stats_;
    }

private:
    struct Pending {
        const ::prag::TokenChunk* tokens;
        std::uint32_t k, nprobe;
        std::promise<::prag::RetrievalOutcome> result;
    };

    void run() {
        for (;;) {
            std::vector<Pending> batch;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [this] { return stop_ || !queue_.empty(); });
                if (queue_.empty()) return;  // stop_ and drained
                const std::uint32_t k = queue_.front().k, nprobe = queue_.front().nprobe;
                for (auto it = queue_.begin(); it != queue_.end() && batch.size() < max_batch_;) {
                    if (it->k == k && it->nprobe == nprobe) {
                        batch.push_back(std::move(*it));
                        it = queue_.erase(it);
                    } else {
                        ++it;
                    }
                }
                stats_.requests += batch.size();
                stats_.batches += 1;
                stats_.max_batch_seen = std::max<std::uint64_t>(stats_.max_batch_seen, batch.size());
            }
            std::vector<const ::prag::TokenChunk*> qs;
            qs.reserve(batch.size());
            for (const auto& p : batch) qs.push_back(p.tokens);
            try {
                auto outs = gpu_->retrieve_batch(qs, batch[0].k, batch[0].nprobe);
                for (std::size_t i = 0; i < batch.size(); ++i) batch[i].result.set_value(std::move(outs[i]));
            } catch (...) {
                for (auto& p : batch) p.result.set_exception(std::current_exception());
            }
        }
    }

    GpuRetriever* gpu_;
    std::uint32_t max_batch_;
    mutable std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Pending> queue_;
    bool stop_ = false;
    Stats stats_;
    std::thread worker_;
};

// Drop-in for prag::RetrievalService (service.hpp:243-362): same constructor
// arguments (plus the CUDA device and the batch cap), same start/port/stop,
// same frames and error behaviour, GPU batched retrieval behind it.
class GpuRetrievalService {
public:
    GpuRetrievalService(const ::prag::Database& db, const ::prag::IvfIndex& index,
                        const ::prag::PqCodebook& codebook, std::uint64_t embed_seed,
                        ::prag::RetrievalPerfModel perf = {}, double safety_margin = 0.10, int device = 0,
                        std::uint32_t max_batch = 64)
        : gpu_(db, index, codebook, embed_seed, perf, safety_margin, device), batcher_(gpu_, max_batch) {}

    ~GpuRetrievalService() { stop(); }

    std::uint16_t start(const std::string& address = "127.0.0.1", std::uint16_t port = 0) {
        listen_fd_ = ::socket(AF_INET, SOCK_STREAM, 0);
        if (listen_fd_ < 0) throw ConfigError("service: socket() failed");
        int one = 1;
        ::setsockopt(listen_fd_, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
        sockaddr_in addr{};
        addr.sin_family = AF_INET;
        addr.sin_port = htons(port);
        if (::inet_pton(AF_INET, address.c_str(), &addr.sin_addr) != 1)
            throw ConfigError("service: invalid bind address " + address);
        if (::bind(listen_fd_, reinterpret_cast<sockaddr*>(&addr), sizeof(addr)) != 0)
            throw ConfigError("service: bind failed on " + address + ":" + std::to_string(port));
        if (::listen(listen_fd_, 64) != 0) throw ConfigError("service: listen failed");
        socklen_t len = sizeof(addr);
        ::getsockname(listen_fd_, reinterpret_cast<sockaddr*>(&addr), &len);
        port_ = ntohs(addr.sin_port);
        running_ = true;
        acceptor_ = std::thread([this] {
            while (running_) {
                const int fd = ::accept(listen_fd_, nullptr, nullptr);
                if (fd < 0) break;
                int nd = 1;
                ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &nd, sizeof(nd));
                std::lock_guard<std::mutex> lk(conn_mu_);
                conns_.insert(fd);
                workers_.emplace_back([this, fd] { serve(fd); });
            }
        });
        return port_;
    }

    std::uint16_t port() const { return port_; }
    GpuRetriever& retriever() { return gpu_; }
    BatchingRetriever::Stats batch_stats() const { return batcher_.stats(); }

    void stop() {
        if (!running_.exchange(false)) return;
        ::shutdown(listen_fd_, SHUT_RDWR);
        ::close(listen_fd_);
        {
            std::lock_guard<std::mutex> lk(conn_mu_);
            for (int fd : conns_) ::shutdown(fd, SHUT_RDWR);
        }
        if (acceptor_.joinable()) acceptor_.join();
        for (auto& t : workers_)
            if (t.joinable()) t.join();
        workers_.clear();
    }

private:
    // One connection: frames in, frames out (service.hpp:307-350 semantics).
    void serve(int fd) {
        using ::prag::detail::read_exact;
        using ::prag::detail::send_frame;
        for (bool open = true; open;) {
            char magic[8];
            if (read_exact(fd, magic, 8) != 0) break;
            if (std::memcmp(magic, ::prag::kWireMagic, 8) != 0) {
                // same protocol name, other version: framing is lost for good
                const bool skew = std::memcmp(magic, ::prag::kWireMagic, 7) == 0;
                send_frame(fd, ::prag::kMsgError,
                           ::prag::encode_error({skew ? ::prag::kErrBadVersion : ::prag::kErrBadMagic,
                                                 skew ? "unsupported protocol version" : "bad frame magic"}));
                if (skew) break;
                continue;
            }
            std::uint32_t n = 0;
            if (read_exact(fd, &n, 4) != 0) break;
            if (n < 1 || n > ::prag::kMaxFrameLen) {
                send_frame(fd, ::prag::kMsgError, ::prag::encode_error({::prag::kErrBadPayload, "bad frame length"}));
                break;
            }
            std::vector<std::uint8_t> body(n);
            if (read_exact(fd, body.data(), n) != 0) break;
            if (body[0] != ::prag::kMsgRequest) {
                send_frame(fd, ::prag::kMsgError,
                           ::prag::encode_error({::prag::kErrBadType, "unexpected message type"}));
                continue;
            }
            try {
                const auto req = ::prag::decode_request(std::vector<std::uint8_t>(body.begin() + 1, body.end()));
                ::prag::Stopwatch clock;
                auto outcome = batcher_.retrieve(req.query_tokens, req.k, req.directive);
                ::prag::RetrievalResponse resp;
                resp.request_id = req.request_id;
                resp.nprobe_used = outcome.nprobe_used;
                resp.server_latency_s = clock.elapsed_s();
                resp.neighbors = std::move(outcome.neighbors);
                open = send_frame(fd, ::prag::kMsgResponse, ::prag::encode_response(resp));
            } catch (const std::exception& e) {
                send_frame(fd, ::prag::kMsgError, ::prag::encode_error({::prag::kErrBadPayload, e.what()}));
            }
        }
        ::close(fd);
        std::lock_guard<std::mutex> lk(conn_mu_);
        conns_.erase(fd);
    }

    GpuRetriever gpu_;
    BatchingRetriever batcher_;
    int listen_fd_ = -1;
    std::uint16_t port_ = 0;
    std::atomic<bool> running_{false};
    std::thread acceptor_;
    std::vector<std::thread> workers_;
    std::mutex conn_mu_;
    std::set<int> conns_;
};

}  // namespace gpu
}  // namespace prag
