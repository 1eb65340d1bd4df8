// Fixed worker pool for host-side staging (the transfer stage's CPU part:
// copying tile windows out of the caller's images into pinned staging).
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace qrm {

class HostPool {
public:
    explicit HostPool(int threads, std::function<void()> init = {}) {
        for (int i = 0; i < threads; ++i)
            workers_.emplace_back([this, init] {
                if (init) init();  // e.g. pin the worker to the GPU's NUMA node
                loop();
            });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    int size() const { return static_cast<int>(workers_.size()); }

    // fn(begin, end) over [0, n) in chunks; the calling thread helps.
    void parallel_for(int64_t n, int64_t chunk, const std::function<void(int64_t, int64_t)>& fn) {
        if (n <= 0) return;
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            n_ = n;
            chunk_ = chunk > 0 ? chunk : 1;
            next_.store(0);
            active_ = static_cast<int>(workers_.size());
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return active_ == 0; });
        fn_ = nullptr;
    }

private:
    void work() {
        while (true) {
            const int64_t b = next_.fetch_add(chunk_);
            if (b >= n_) break;
            (*fn_)(b, b + chunk_ < n_ ? b + chunk_ : n_);
        }
    }
    void loop() {
        uint64_t seen = 0;
        while (true) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            work();
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--active_ == 0) done_cv_.notify_all();
            }
        }
    }

    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int64_t, int64_t)>* fn_ = nullptr;
    int64_t n_ = 0, chunk_ = 1;
    std::atomic<int64_t> next_{0};
    int active_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

}  // namespace qrm
