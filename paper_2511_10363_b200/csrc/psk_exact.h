// psk_exact.h -- host interface of the exact and fast device paths.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "psk_common.cuh"
#include "psk_plan.hpp"

namespace psk {

// Per-device, per-kernel launch setup, done once: raise the kernel's dynamic
// shared-memory limit to `smem` and return its co-resident CTAs per SM
// (cudaFuncSetAttribute / the occupancy query cost microseconds per call,
// which showed as idle gaps between the short kernels of a small-T run).
template <class Kernel>
int kernel_setup(Kernel kernel, int block, int smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), dev, block, smem);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
  cache[key] = per_sm;
  return per_sm;
}
// Chunk length floor of a Sequential chunk scan (psk_alg 0: one chain of
// combines over the chunk elements, scan.hpp:198-210): the chain costs one
// combine latency per chunk and each per-step walk one step latency per step
// of a chunk, so about sqrt(T) chunks of sqrt(T) steps balance the two
// (T = 2^14: 59 ms with 16384 one-step chunks, profiles/r02_v3/csv).
inline long long seq_chunk_floor(long long T) {
  long long s = 1;
  while (s * s < T) s <<= 1;  // power-of-two bracket, then refine
  long long lo = s >> 1;
  while (lo * lo < T) ++lo;
  return lo < 1 ? 1 : lo;
}

inline int device_sms() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return cache[dev] = sms > 0 ? sms : 148;
}

// Launch bookkeeping shared by all paths: the stream, the device error word,
// a launch counter and optional per-kernel CUDA-event timing.
struct ExactLaunch {
  cudaStream_t stream = nullptr;
  unsigned* err = nullptr;
  long long launches = 0;
  bool profile = false;
  std::vector<const char*> names;
  std::vector<cudaEvent_t> evs;  // evs[0] = start; kernel i ends at evs[i+1]
  // async mode: the event spans of calls not yet synchronised
  std::vector<std::pair<std::vector<cudaEvent_t>, std::vector<const char*>>> pending;
  // optional DLB phase trace of this context (option "dlb_trace"; stamps of
  // every scan are appended to trace_path, read by tools/dlb_trace.py)
  unsigned long long* dlb_trace = nullptr;
  long long dlb_trace_cap = 0;  // tiles
  std::string dlb_trace_path;
  void start(bool keep = false) {
    launches = 0;
    if (keep && !evs.empty()) {
      pending.emplace_back(std::move(evs), std::move(names));
    } else {
      for (auto e : evs) cudaEventDestroy(e);
    }
    evs.clear();
    names.clear();
    if (!profile) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, stream);
    evs.push_back(e);
  }
  // called right after each kernel launch (launches on one stream are
  // serialised, so kernel i spans evs[i] .. evs[i+1])
  // a profiled span that is not a kernel launch (host <-> device copies)
  void mark(const char* name) {
    if (!profile) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, stream);
    evs.push_back(e);
    names.push_back(name);
  }
  void count(const char* name) {
    ++launches;
    if (!profile) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, stream);
    evs.push_back(e);
    names.push_back(name);
  }
};

// method: 0 = PKF, 1 = PRTS, 2 = PTFS
template <typename S>
void exact_run(ExactLaunch& L, const ModelView<S>& m, int method,
               const ScanPlan& plan, S* el0, S* el1, S* el2, S* bel0, S* mean,
               S* cov);

// fast path: returns false when (nx, ny) has no compiled instantiation
struct FastArgs {
  int method = 0;       // 0 PKF, 1 PRTS, 2 PTFS
  int alg = 3;          // psk_alg
  unsigned long long sengupta_n = 1;
  long long chunk = 32;
  int waves = 0;        // auto chunk (chunk = 0): whole waves of chunks (0: default)
  int tile = 1;         // dims > 4: register-tiled kernels where instantiated (psk_tile*.cuh)
};
template <typename S>
bool fast_supported(int nx, int ny);
template <typename S>
int fast_run(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a,
             S* mean, S* cov, void* (*alloc)(size_t, void*), void* alloc_ctx);

// wide fast path (psk_wide_impl.cuh): runtime nx, ny <= 16, PKF and PRTS;
// returns -1 when the request is not covered (PTFS -> exact path)
template <typename S>
int wide_run(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a, S* mean, S* cov,
             void* (*alloc)(size_t, void*), void* alloc_ctx);

// register-tiled warp kernels for compile-time (nx, ny) (psk_tile_impl.cuh);
// -1 when the request has no instantiation (then the wide path runs)
template <typename S>
int tile_run(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a, S* mean, S* cov,
             void* (*alloc)(size_t, void*), void* alloc_ctx);

// PTFS with forward (A) and backward (B) passes on two contexts
template <typename S>
int fast_ptfs2(ExactLaunch& LA, const ModelView<S>& mA, int devA, ExactLaunch& LB,
               const ModelView<S>& mB, int devB, const FastArgs& a, S* mean, S* cov,
               void* (*allocA)(size_t, void*), void* ctxA, void* (*allocB)(size_t, void*),
               void* ctxB);

template <typename S>
int fast_shard_phase(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a, int phase,
                     void** scratch, S* mean, S* cov, const S* carry, S* elem_out,
                     void* (*alloc)(size_t, void*), void* actx, const S* fmean = nullptr,
                     const S* fcov = nullptr);
template <typename S>
void fast_shard_release(void* scratch);
template <typename S>
int fast_fold(ExactLaunch& L, int kind, int nx, const S* aggs, int count, S* out);

}  // namespace psk
