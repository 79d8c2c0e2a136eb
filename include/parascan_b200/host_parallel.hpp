// host_parallel.hpp -- the host-side worker split of the C++ shim's
// marshalling (cuda_backend.hpp) and of gen_model_par (model_gen_par.hpp).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

namespace parascan {
namespace psk_detail {

// worker count: $PSK_HOST_THREADS, else the hardware concurrency
inline unsigned host_threads() {
  if (const char* e = std::getenv("PSK_HOST_THREADS")) {
    const long v = std::strtol(e, nullptr, 10);
    if (v >= 1) return unsigned(v);
  }
  const unsigned h = std::thread::hardware_concurrency();
  return h ? h : 1;
}

// fn(lo, hi) over [0, n) in contiguous ranges of at least `grain` steps
template <class Fn>
void parallel_for(std::size_t n, std::size_t grain, Fn&& fn) {
  const std::size_t want = grain ? (n + grain - 1) / grain : 1;
  const std::size_t nt = std::max<std::size_t>(1, std::min<std::size_t>(host_threads(), want));
  if (nt <= 1) {
    fn(std::size_t(0), n);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(nt - 1);
  std::exception_ptr err;
  std::mutex mu;
  auto body = [&](std::size_t i) {
    try {
      fn(n * i / nt, n * (i + 1) / nt);
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu);
      if (!err) err = std::current_exception();
    }
  };
  for (std::size_t i = 1; i < nt; ++i) pool.emplace_back(body, i);
  body(0);
  for (auto& t : pool) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace psk_detail
}  // namespace parascan
