// pool.hpp -- tiny fork/join thread pool for the host dependency builder.
// run(f) executes f(0..n-1) with the calling thread as worker 0 and returns
// when all have finished.  Workers spin on a generation counter for a while
// after each job (waking a sleeping thread costs milliseconds on the KVM
// hosts this runs on, more than a whole 1M-task build), then sleep on a
// condition variable.  The caller spins for completion.
#pragma once
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

// Deliberately NOT the x86 PAUSE instruction: under KVM, pause-loop exiting
// deschedules a spinning vCPU (measured: ~4 ms per worker per fork/join).
#define BT_CPU_RELAX() asm volatile("" ::: "memory")

namespace bt {

class Pool {
 public:
  explicit Pool(int n, int spin_us = 5000) : n_(n < 1 ? 1 : n), spin_us_(spin_us) {
    for (int i = 1; i < n_; ++i) threads_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_.store(true, std::memory_order_relaxed);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    for (auto &t : threads_) t.join();
  }
  int size() const { return n_; }

  void run(const std::function<void(int)> &f) {
    if (n_ == 1) {
      f(0);
      return;
    }
    job_ = &f;
    pending_.store(n_ - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> g(m_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    if (sleepers_.load(std::memory_order_acquire) > 0) cv_.notify_all();
    f(0);
    while (pending_.load(std::memory_order_acquire) != 0) BT_CPU_RELAX();
    job_ = nullptr;
  }

 private:
  void loop(int id) {
    uint64_t seen = 0;   // the generation at construction (a late-starting thread must not skip a job)
    for (;;) {
      // spin for a new generation, then sleep
      uint64_t g = gen_.load(std::memory_order_acquire);
      if (g == seen) {
        const auto until = std::chrono::steady_clock::now() + std::chrono::microseconds(spin_us_);
        for (unsigned it = 0;; ++it) {
          BT_CPU_RELAX();
          g = gen_.load(std::memory_order_acquire);
          if (g != seen) break;
          if ((it & 1023) == 1023 && std::chrono::steady_clock::now() > until) {
            std::unique_lock<std::mutex> l(m_);
            sleepers_.fetch_add(1, std::memory_order_acq_rel);
            cv_.wait(l, [&] { return gen_.load(std::memory_order_acquire) != seen; });
            sleepers_.fetch_sub(1, std::memory_order_acq_rel);
            g = gen_.load(std::memory_order_acquire);
            break;
          }
        }
      }
      seen = g;
      if (stop_.load(std::memory_order_relaxed)) return;
      (*job_)(id);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }

  int n_;
  int spin_us_;
  std::vector<std::thread> threads_;
  std::mutex m_;
  std::condition_variable cv_;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> sleepers_{0};
  std::atomic<bool> stop_{false};
  const std::function<void(int)> *job_ = nullptr;
  std::atomic<int> pending_{0};
};

}  // namespace bt
