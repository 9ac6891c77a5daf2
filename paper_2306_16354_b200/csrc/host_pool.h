// host_pool.h — persistent host worker threads for the pipeline's host-side
// parallel loops (the dendrogram fold, the cut, output copy-out, page
// pre-faulting).  Spawning a fresh std::thread set for every loop of every
// call made the dendrogram stage jitter between steps; the workers here are
// created once (hardware_concurrency - 1, at most 31) and sleep between
// batches.
//
//   HostPool::get().run(ntasks, fn)      fn(task) for task in [0, ntasks), caller helps
//   auto b = HostPool::get().submit(...); ...; b.wait()   start now, join later
//
// One batch runs at a time (a mutex serialises callers); tasks must not throw.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace slk {

class HostPool {
  public:
    static HostPool &get() {
        static HostPool pool;
        return pool;
    }
    int workers() const { return (int)threads_.size(); }

    class Batch {
      public:
        explicit Batch(HostPool *p) : p_(p) {}
        Batch(Batch &&o) noexcept : p_(o.p_) { o.p_ = nullptr; }
        Batch &operator=(Batch &&o) noexcept {
            if (this != &o) {
                wait();
                p_ = o.p_;
                o.p_ = nullptr;
            }
            return *this;
        }
        Batch(const Batch &) = delete;
        ~Batch() { wait(); }
        void wait() {
            if (!p_) return;
            p_->drain();  // the caller helps
            {
                std::unique_lock<std::mutex> lk(p_->mu_);
                // every task done and no worker still inside this batch's drain
                p_->done_cv_.wait(lk, [&] { return p_->remaining_.load() == 0 && p_->active_ == 0; });
                p_->fn_ = nullptr;
            }
            p_->batch_mu_.unlock();
            p_ = nullptr;
        }

      private:
        HostPool *p_;
    };

    Batch submit(int ntasks, std::function<void(int)> fn) {
        batch_mu_.lock();  // released by Batch::wait
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = std::move(fn);
            ntasks_ = ntasks;
            next_.store(0);
            remaining_.store(ntasks);
            gen_++;
        }
        cv_.notify_all();
        return Batch(this);
    }
    void run(int ntasks, std::function<void(int)> fn) { submit(ntasks, std::move(fn)).wait(); }

  private:
    HostPool() {
        const unsigned hc = std::thread::hardware_concurrency();
        const int n = (int)std::min(31u, std::max(1u, hc) - 1u);
        for (int i = 0; i < n; i++) threads_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : threads_) t.join();
    }
    void loop() {
        uint64_t seen = 0;
        while (true) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                active_++;
            }
            drain();
            {
                std::lock_guard<std::mutex> lk(mu_);
                active_--;
            }
            done_cv_.notify_all();
        }
    }
    void drain() {
        std::function<void(int)> *f = &fn_;
        const int nt = ntasks_;
        for (int t; (t = next_.fetch_add(1)) < nt;) {
            (*f)(t);
            if (remaining_.fetch_sub(1) == 1) {
                std::lock_guard<std::mutex> lk(mu_);
                done_cv_.notify_all();
            }
        }
    }

    std::vector<std::thread> threads_;
    std::mutex mu_, batch_mu_;
    std::condition_variable cv_, done_cv_;
    std::function<void(int)> fn_;
    int ntasks_ = 0, active_ = 0;
    std::atomic<int> next_{0}, remaining_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// body(lo, hi) over [0, n) in `parts` contiguous slices on the pool
template <class F>
void pool_slices(int64_t n, int parts, F body) {
    parts = (int)std::max<int64_t>(1, std::min<int64_t>(parts, n));
    HostPool::get().run(parts, [&](int k) { body(n * k / parts, n * (k + 1) / parts); });
}

}  // namespace slk
