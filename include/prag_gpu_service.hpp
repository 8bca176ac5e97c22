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

#include <poll.h>
#include <sys/eventfd.h>

#include <cerrno>
#include <condition_variable>
#include <deque>
#include <future>
#include <map>
#include <set>

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

// Client connections of a GpuRetrievalService: one handler thread per
// socket. shut() wakes every handler blocked in a read (the socket stays
// open until its handler closes it); join() waits for all of them.
class ConnectionRegistry {
public:
    template <class Handler>
    void spawn(int fd, Handler handler) {
        std::lock_guard<std::mutex> lk(mu_);
        open_.insert(fd);
        threads_.emplace_back([this, fd, handler] {
            handler(fd);
            {
                std::lock_guard<std::mutex> g(mu_);
                open_.erase(fd);
            }
            ::close(fd);
        });
    }
    void shut() {
        std::lock_guard<std::mutex> lk(mu_);
        for (int fd : open_) ::shutdown(fd, SHUT_RDWR);
    }
    void join() {
        std::vector<std::thread> ts;
        {
            std::lock_guard<std::mutex> lk(mu_);
            ts.swap(threads_);
        }
        for (auto& t : ts) t.join();
    }

private:
    std::mutex mu_;
    std::set<int> open_;
    std::vector<std::thread> threads_;
};

// Drop-in for prag::RetrievalService (service.hpp:243-362): same constructor
// arguments (plus the CUDA device and the batch cap), same start/port/stop
// contract and bind errors, same frames and error behaviour; GPU batched
// retrieval behind it. The acceptor polls the listening socket together with
// an eventfd, so stop() wakes it by writing the eventfd rather than by
// tearing the listening socket down under a blocked accept().
class GpuRetrievalService {
public:
    GpuRetrievalService(const ::prag::Database& db, const ::prag::IvfIndex& index,
                        const ::prag::PqCodebook& codebook, std::uint64_t embed_seed,
                        ::prag::RetrievalPerfModel perf = {}, double safety_margin = 0.10, int device = 0,
                        std::uint32_t max_batch = 64)
        : gpu_(db, index, codebook, embed_seed, perf, safety_margin, device), batcher_(gpu_, max_batch) {}

    ~GpuRetrievalService() { stop(); }

    // Listens on address:port (0 = ephemeral); returns the bound port.
    std::uint16_t start(const std::string& address = "127.0.0.1", std::uint16_t port = 0) {
        const Listener l = bind_listener(address, port);
        wake_fd_ = ::eventfd(0, EFD_CLOEXEC);
        if (wake_fd_ < 0) {
            ::close(l.fd);
            throw ConfigError("service: eventfd() failed");
        }
        listen_fd_ = l.fd;
        port_ = l.port;
        acceptor_ = std::thread([this] { acceptor_main(); });
        return port_;
    }

    std::uint16_t port() const { return port_; }
    GpuRetriever& retriever() { return gpu_; }
    BatchingRetriever::Stats batch_stats() const { return batcher_.stats(); }

    // Idempotent: wakes and joins the acceptor, then ends every connection.
    void stop() {
        if (!acceptor_.joinable()) return;
        const std::uint64_t one = 1;
        (void)!::write(wake_fd_, &one, sizeof one);
        acceptor_.join();
        ::close(listen_fd_);
        ::close(wake_fd_);
        listen_fd_ = wake_fd_ = -1;
        conns_.shut();
        conns_.join();
    }

private:
    struct Listener {
        int fd;
        std::uint16_t port;
    };

    // socket/bind/listen with the reference's ConfigError texts
    // (service.hpp:254-268 behaviour).
    static Listener bind_listener(const std::string& address, std::uint16_t port) {
        in_addr ip{};
        if (::inet_pton(AF_INET, address.c_str(), &ip) != 1)
            throw ConfigError("service: invalid bind address " + address);
        const int fd = ::socket(AF_INET, SOCK_STREAM | SOCK_CLOEXEC, 0);
        if (fd < 0) throw ConfigError("service: socket() failed");
        auto fail = [fd](const std::string& what) {
            ::close(fd);
            throw ConfigError(what);
        };
        const int on = 1;
        ::setsockopt(fd, SOL_SOCKET, SO_REUSEADDR, &on, sizeof on);
        sockaddr_in want{};
        want.sin_family = AF_INET;
        want.sin_addr = ip;
        want.sin_port = htons(port);
        if (::bind(fd, reinterpret_cast<const sockaddr*>(&want), sizeof want) != 0)
            fail("service: bind failed on " + address + ":" + std::to_string(port));
        if (::listen(fd, SOMAXCONN) != 0) fail("service: listen failed");
        sockaddr_in got{};
        socklen_t n = sizeof got;
        ::getsockname(fd, reinterpret_cast<sockaddr*>(&got), &n);
        return {fd, ntohs(got.sin_port)};
    }

    void acceptor_main() {
        pollfd pf[2] = {{listen_fd_, POLLIN, 0}, {wake_fd_, POLLIN, 0}};
        while (true) {
            if (::poll(pf, 2, -1) < 0) {
                if (errno == EINTR) continue;
                return;
            }
            if (pf[1].revents) return;  // stop()
            if (!(pf[0].revents & POLLIN)) continue;
            const int fd = ::accept4(listen_fd_, nullptr, nullptr, SOCK_CLOEXEC);
            if (fd < 0) continue;  // the peer went away before accept
            const int on = 1;
            ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &on, sizeof on);
            conns_.spawn(fd, [this](int c) { serve(c); });
        }
    }

    static bool send_error(int fd, std::uint32_t code, const std::string& what) {
        return ::prag::detail::send_frame(fd, ::prag::kMsgError, ::prag::encode_error({code, what}));
    }

    // What one read of the connection produced (service.hpp:307-350 semantics).
    enum class Got { Closed, Skip, Drop, Request };

    static Got next_request(int fd, ::prag::RetrievalRequest* req) {
        using ::prag::detail::read_exact;
        char head[8];
        if (read_exact(fd, head, sizeof head) != 0) return Got::Closed;
        if (std::memcmp(head, ::prag::kWireMagic, sizeof head) != 0) {
            // a different version of the same protocol: framing is lost
            const bool version_skew = std::memcmp(head, ::prag::kWireMagic, 7) == 0;
            if (version_skew) {
                send_error(fd, ::prag::kErrBadVersion, "unsupported protocol version");
                return Got::Drop;
            }
            send_error(fd, ::prag::kErrBadMagic, "bad frame magic");
            return Got::Skip;
        }
        std::uint32_t len = 0;
        if (read_exact(fd, &len, sizeof len) != 0) return Got::Closed;
        if (len == 0 || len > ::prag::kMaxFrameLen) {
            send_error(fd, ::prag::kErrBadPayload, "bad frame length");
            return Got::Drop;
        }
        std::vector<std::uint8_t> frame(len);
        if (read_exact(fd, frame.data(), len) != 0) return Got::Closed;
        if (frame.front() != ::prag::kMsgRequest) {
            send_error(fd, ::prag::kErrBadType, "unexpected message type");
            return Got::Skip;
        }
        try {
            *req = ::prag::decode_request(std::vector<std::uint8_t>(frame.begin() + 1, frame.end()));
        } catch (const std::exception& e) {
            send_error(fd, ::prag::kErrBadPayload, e.what());
            return Got::Skip;
        }
        return Got::Request;
    }

    void serve(int fd) {
        for (;;) {
            ::prag::RetrievalRequest req;
            const Got got = next_request(fd, &req);
            if (got == Got::Closed || got == Got::Drop) return;
            if (got == Got::Skip) continue;
            ::prag::RetrievalResponse resp;
            resp.request_id = req.request_id;
            try {
                ::prag::Stopwatch timer;
                auto out = batcher_.retrieve(req.query_tokens, req.k, req.directive);
                resp.server_latency_s = timer.elapsed_s();
                resp.nprobe_used = out.nprobe_used;
                resp.neighbors = std::move(out.neighbors);
            } catch (const std::exception& e) {
                send_error(fd, ::prag::kErrBadPayload, e.what());
                continue;
            }
            if (!::prag::detail::send_frame(fd, ::prag::kMsgResponse, ::prag::encode_response(resp))) return;
        }
    }

    GpuRetriever gpu_;
    BatchingRetriever batcher_;
    int listen_fd_ = -1, wake_fd_ = -1;
    std::uint16_t port_ = 0;
    std::thread acceptor_;
    ConnectionRegistry conns_;
};

}  // namespace gpu
}  // namespace prag
