// host_pool.hpp — a small persistent host thread pool (plain C++; used by the multi-device host
// path csrc/multi.cu and the C++ shim's batch packing).
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace dcat {

// Persistent host workers: run(n, f) calls f(0 .. n-1) on the workers and
// the calling thread and returns when all are done. Jobs from several threads are serialised.
// (Spawning std::threads per phase cost ~20-50 us each, several ms per call at 16 threads.)
class ThreadPool {
public:
    explicit ThreadPool(unsigned workers) {
        for (unsigned i = 0; i < workers; i++) th_.emplace_back([this] { loop(); });
    }
    ~ThreadPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    unsigned size() const { return static_cast<unsigned>(th_.size()) + 1; }
    void run(unsigned n, const std::function<void(unsigned)>& f) {
        if (n == 0) return;
        if (n == 1 || th_.empty()) {
            for (unsigned i = 0; i < n; i++) f(i);
            return;
        }
        std::lock_guard<std::mutex> job(job_m_);
        {
            // no worker of the previous job is still taking items when the counter resets
            std::unique_lock<std::mutex> lk(m_);
            idle_cv_.wait(lk, [&] { return active_ == 0; });
            f_ = &f;
            n_ = n;
            next_.store(0);
            done_ = 0;
            gen_++;
        }
        cv_.notify_all();
        take(&f, n);
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [&] { return done_ == n; });
        f_ = nullptr;
    }

private:
    void take(const std::function<void(unsigned)>* f, unsigned n) {
        unsigned k = 0, mine = 0;
        while ((k = next_.fetch_add(1)) < n) {
            (*f)(k);
            mine++;
        }
        if (mine) {
            std::lock_guard<std::mutex> lk(m_);
            done_ += mine;
            if (done_ == n) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(unsigned)>* f = nullptr;
            unsigned n = 0;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || (gen_ != seen && f_ != nullptr); });
                if (stop_) return;
                seen = gen_;
                f = f_;
                n = n_;
                active_++;
            }
            take(f, n);
            std::lock_guard<std::mutex> lk(m_);
            if (--active_ == 0) idle_cv_.notify_all();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_, job_m_;
    std::condition_variable cv_, done_cv_, idle_cv_;
    const std::function<void(unsigned)>* f_ = nullptr;
    unsigned n_ = 0, done_ = 0, active_ = 0;
    std::atomic<unsigned> next_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
};

}  // namespace dcat
