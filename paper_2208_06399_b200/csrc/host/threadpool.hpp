// Small persistent host thread pool: parallel_for over task indices, and a
// background "job" runner so batch staging overlaps the GPU step.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace asb {

class ThreadPool {
 public:
  explicit ThreadPool(unsigned n = 0) {
    if (n == 0) n = std::max(1u, std::thread::hardware_concurrency());
    for (unsigned i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
  }
  ~ThreadPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  unsigned size() const { return static_cast<unsigned>(th_.size()); }

  // Runs fn(i) for i in [0, n) on the pool (the caller helps); returns when done.
  void parallel_for(int64_t n, const std::function<void(int64_t)>& fn) {
    if (n <= 0) return;
    std::atomic<int64_t> next{0};
    std::atomic<int64_t> done{0};
    auto body = [&] {
      for (int64_t i; (i = next.fetch_add(1)) < n;) {
        fn(i);
        done.fetch_add(1);
      }
    };
    const unsigned helpers = static_cast<unsigned>(std::min<int64_t>(n - 1, th_.size()));
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (unsigned h = 0; h < helpers; ++h) q_.push_back(body);
    }
    cv_.notify_all();
    body();
    while (done.load() < n) std::this_thread::yield();
    // helpers may still be returning from body(); wait until they leave it
    std::unique_lock<std::mutex> lk(mu_);
    idle_cv_.wait(lk, [&] { return running_ == 0 && q_.empty(); });
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
        if (stop_ && q_.empty()) return;
        job = std::move(q_.back());
        q_.pop_back();
        ++running_;
      }
      job();
      {
        std::lock_guard<std::mutex> lk(mu_);
        --running_;
      }
      idle_cv_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::vector<std::function<void()>> q_;
  std::mutex mu_;
  std::condition_variable cv_, idle_cv_;
  int running_ = 0;
  bool stop_ = false;
};

// Process-wide pool for batch staging (one per process is enough: contexts
// of one process run one host thread per device).
ThreadPool& staging_pool();

}  // namespace asb
