// Host-side staging for pageable operands (the reference's NumPy arrays,
// matmul.py:342-366): a parallel 2-D memcpy between pageable and pinned host
// memory, run by a small persistent thread pool so the k-phased H2D / compute /
// D2H pipeline can feed the GPU from pageable memory at the host's copy rate.
// Host code only; no kernels.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace paco {
namespace {

struct CopyJob {
  char* dst;
  const char* src;
  int64_t dpitch, spitch, width, rows;
  int parts;
};

class StagePool {
 public:
  static StagePool& get() {
    static StagePool* p = new StagePool();  // never destroyed: workers may outlive static teardown
    return *p;
  }

  // Copy with `threads` participants (the caller is one of them).  A worker
  // joins a job only while it is open, under the lock run() opens and closes
  // it with; run() closes the job once every part is done and no worker is
  // inside.  So a worker that wakes late -- after its job finished -- finds it
  // closed and takes nothing: it can never pair an old job's pointers with the
  // part counter of the next job (which would mark a part done that nobody
  // copied, and write into the old job's buffers).
  void run(const CopyJob& job, int threads) {
    std::lock_guard<std::mutex> serial(call_mu_);  // one job at a time
    ensure_workers(threads - 1);
    {
      std::lock_guard<std::mutex> lock(mu_);
      job_ = job;
      next_.store(0);
      done_.store(0);
      ++gen_;
      active_ = threads - 1;
      open_ = true;
    }
    cv_.notify_all();
    work(job);
    std::unique_lock<std::mutex> lock(mu_);
    done_cv_.wait(lock, [&] { return done_.load() == job.parts && inside_ == 0; });
    open_ = false;
  }

 private:
  void ensure_workers(int want) {
    while (int(workers_.size()) < want) {
      const int id = int(workers_.size());
      workers_.emplace_back([this, id] { loop(id); });
      workers_.back().detach();
    }
  }

  void loop(int id) {
    uint64_t seen = 0;
    for (;;) {
      CopyJob j;
      {
        std::unique_lock<std::mutex> lock(mu_);
        cv_.wait(lock, [&] { return gen_ != seen; });
        seen = gen_;
        if (!open_ || id >= active_) continue;  // finished already, or not a participant
        j = job_;
        ++inside_;
      }
      work(j);
      {
        std::lock_guard<std::mutex> lock(mu_);
        --inside_;
      }
      done_cv_.notify_all();
    }
  }

  void work(const CopyJob& j) {
    for (;;) {
      const int p = next_.fetch_add(1);
      if (p >= j.parts) break;
      const int64_t r0 = j.rows * p / j.parts, r1 = j.rows * (p + 1) / j.parts;
      if (j.dpitch == j.width && j.spitch == j.width) {
        memcpy(j.dst + r0 * j.width, j.src + r0 * j.width, size_t((r1 - r0) * j.width));
      } else {
        for (int64_t r = r0; r < r1; ++r) memcpy(j.dst + r * j.dpitch, j.src + r * j.spitch, size_t(j.width));
      }
      if (done_.fetch_add(1) + 1 == j.parts) {
        std::lock_guard<std::mutex> lock(mu_);
        done_cv_.notify_all();
      }
    }
  }

  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> workers_;
  CopyJob job_{};
  std::atomic<int> next_{0}, done_{0};
  uint64_t gen_ = 0;
  int active_ = 0;
  int inside_ = 0;
  bool open_ = false;
};

}  // namespace
}  // namespace paco

extern "C" int paco_host_copy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                                int64_t rows, int threads) {
  using namespace paco;
  if (rows <= 0 || width <= 0) return PACO_OK;
  if (!dst || !src || dpitch < width || spitch < width) {
    set_error("paco_host_copy2d: bad pointers or pitches");
    return PACO_ERR_ARG;
  }
  threads = std::max(1, std::min(threads, 64));
  const int64_t bytes = width * rows;
  // ~1 MiB per part, at least one part per participant for big copies
  int parts = int(std::min<int64_t>(rows, std::max<int64_t>(1, bytes >> 20)));
  parts = std::max(parts, std::min<int>(threads, int(rows)));
  if (threads == 1 || parts == 1 || bytes < (int64_t(1) << 20)) {
    for (int64_t r = 0; r < rows; ++r)
      memcpy(static_cast<char*>(dst) + r * dpitch, static_cast<const char*>(src) + r * spitch, size_t(width));
    return PACO_OK;
  }
  CopyJob job{static_cast<char*>(dst), static_cast<const char*>(src), dpitch, spitch, width, rows, parts};
  StagePool::get().run(job, threads);
  return PACO_OK;
}
