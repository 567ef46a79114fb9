// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp header).
//
// A persistent worker pool for the oracle's independent-item loops. Every item
// is computed start to finish by exactly one thread with the serial loop's
// arithmetic, so results are bit-identical for any thread count (the
// reference itself is single-threaded). H2O_THREADS=1 runs
// everything inline on the calling thread.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace h2o {

class WorkerPool {
 public:
  static WorkerPool& get() {
    static WorkerPool p;
    return p;
  }
  int threads() const { return nthreads_; }

  // f(i) for i in [0, n); items handed out dynamically; exceptions rethrown.
  void run(int64_t n, const std::function<void(int64_t)>& f) {
    if (n <= 0) return;
    if (nthreads_ <= 1 || n == 1 || in_pool_) {
      for (int64_t i = 0; i < n; ++i) f(i);
      return;
    }
    std::unique_lock<std::mutex> serial(run_mu_);
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &f;
      n_ = n;
      next_.store(0);
      err_ = nullptr;
      active_ = static_cast<int>(workers_.size());
      ++gen_;
    }
    cv_.notify_all();
    in_pool_ = true;  // nested pool_for calls from inside f run inline
    work(f, n);       // the caller participates
    in_pool_ = false;
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return active_ == 0; });
    job_ = nullptr;
    if (err_) std::rethrow_exception(err_);
  }

  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  WorkerPool() {
    nthreads_ = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    if (const char* e = std::getenv("H2O_THREADS")) nthreads_ = std::max(1, std::atoi(e));
    for (int t = 1; t < nthreads_; ++t) workers_.emplace_back([this] { loop(); });
  }

  void work(const std::function<void(int64_t)>& f, int64_t n) {
    for (int64_t i = next_++; i < n; i = next_++) {
      try {
        f(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu_);
        if (!err_) err_ = std::current_exception();
      }
    }
  }

  void loop() {
    in_pool_ = true;
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int64_t)>* job;
      int64_t n;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
        n = n_;
      }
      if (job) work(*job, n);
      std::lock_guard<std::mutex> g(mu_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }

  int nthreads_ = 1;
  std::vector<std::thread> workers_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int64_t)>* job_ = nullptr;
  int64_t n_ = 0;
  std::atomic<int64_t> next_{0};
  std::exception_ptr err_;
  int active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  static thread_local bool in_pool_;
};

inline thread_local bool WorkerPool::in_pool_ = false;

// Parallel loop over independent items (bit-identical to the serial loop).
template <class F>
inline void pool_for(int64_t n, F&& f) {
  WorkerPool::get().run(n, std::function<void(int64_t)>(std::forward<F>(f)));
}

}  // namespace h2o
