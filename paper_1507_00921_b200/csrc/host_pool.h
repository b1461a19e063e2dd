// A small persistent host thread pool for the complex128 <-> complex64
// conversions of the drop-in entry point (dbp_backpropagate_c128): the
// reference hands the DBP complex128 rows (sigkit.py:56-68) and expects
// complex128 back, so the host casts are part of the call; spread over the
// host cores they overlap the GPU's work on the previous chunk.
#pragma once
#include <algorithm>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace dbp {

class HostPool {
 public:
  explicit HostPool(int threads) {
    for (int i = 1; i < threads; ++i) workers_.emplace_back([this, i] { loop(i); });
    n_ = threads;
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return n_; }
  // fn(lo, hi) over [0, count) split into size() contiguous pieces; the
  // calling thread runs piece 0; returns when every piece is done.  Callers
  // on different threads (plans on different devices sharing the pool) are
  // serialised.
  //
  // Only as many threads take part as the work pays for (`grain` items per
  // piece): waking a sleeping worker costs tens of microseconds, more than
  // converting a few thousand samples on the calling thread.
  void parallel_for(long long count, const std::function<void(long long, long long)>& fn,
                    long long grain = 8192) {
    const int pieces = (int)std::max<long long>(1, std::min<long long>(n_, count / std::max<long long>(1, grain)));
    if (pieces == 1) {
      fn(0, count);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      count_ = count;
      pieces_ = pieces;
      pending_ = pieces - 1;
      ++gen_;
    }
    cv_.notify_all();
    run_piece(0, pieces);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void run_piece(int i, int pieces) {
    const long long per = (count_ + pieces - 1) / pieces;
    const long long lo = std::min<long long>(count_, per * i), hi = std::min<long long>(count_, lo + per);
    if (hi > lo) (*fn_)(lo, hi);
  }
  void loop(int i) {
    unsigned long long seen = 0;
    for (;;) {
      int pieces;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        pieces = pieces_;
      }
      if (i >= pieces) continue;   // this call does not need worker i (the caller waits for pieces - 1)
      run_piece(i, pieces);
      {
        std::lock_guard<std::mutex> g(mu_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(long long, long long)>* fn_ = nullptr;
  long long count_ = 0;
  int pending_ = 0, pieces_ = 1, n_ = 1;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

}  // namespace dbp
