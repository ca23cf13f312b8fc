// Batching of the oracle: the reference's own proj/include/hps/parallel.hpp when it is
// available at build time (oracle/Makefile adds -I/root/reference/proj/include and
// -DHPSO_REFERENCE_HEADERS), else this restatement of it (parallel.hpp:13-58).
// TEST INFRASTRUCTURE ONLY (see hps_oracle.hpp).
#pragma once
#ifdef HPSO_REFERENCE_HEADERS
#include <hps/parallel.hpp>
namespace hpso {
using hps::hardware_workers;
using hps::parallel_for;
}  // namespace hpso
#else
#include <atomic>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

namespace hpso {

inline int hardware_workers() {
  const unsigned hc = std::thread::hardware_concurrency();
  return hc ? int(hc) : 1;
}

template <class Fn>
void parallel_for(int n, int workers, Fn&& fn) {
  if (n <= 0) return;
  const int w = std::min(workers > 0 ? workers : hardware_workers(), n);
  if (w <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int> cursor{0};
  std::atomic<bool> stop{false};
  std::exception_ptr err;
  std::mutex mu;
  auto worker = [&]() {
    while (!stop.load(std::memory_order_relaxed)) {
      const int i = cursor.fetch_add(1, std::memory_order_relaxed);
      if (i >= n) break;
      try {
        fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!err) err = std::current_exception();
        stop.store(true, std::memory_order_relaxed);
      }
    }
  };
  std::vector<std::thread> th;
  th.reserve(w - 1);
  for (int t = 1; t < w; ++t) th.emplace_back(worker);
  worker();
  for (auto& t : th) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace hpso
#endif  // HPSO_REFERENCE_HEADERS
