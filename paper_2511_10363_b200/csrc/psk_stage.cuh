// psk_stage.cuh -- per-thread asynchronous staging of per-step model blocks
// into shared memory (cp.async, LDGSTS), double-buffered.
//
// Every fast-path thread walks its own chunk of consecutive steps, so the
// natural access is "one thread, one contiguous 16..128-byte block per field
// per step".  Issuing the loads for step k+1 before computing step k keeps
// enough bytes in flight to saturate HBM without spending registers (the
// per-step model is 52 scalars = 416 B at nx=4, ny=2, f64).  The shared layout
// is granule-major: granule g of a field for thread t lives at
// base + g * U * NT + t * U (U = 16/8/4 bytes), so a warp's 16-byte reads are
// bank-conflict-free and each thread only ever touches its own granules (no
// block-level barrier is needed -- cp.async.wait_group is per thread).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "psk_mat.cuh"

namespace psk {

template <int BYTES>
struct Gran {
  static constexpr int U = BYTES % 16 == 0 ? 16 : (BYTES % 8 == 0 ? 8 : 4);
  static constexpr int N = BYTES / U;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int U>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
  if constexpr (U == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
  else if constexpr (U == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// A field of BYTES bytes per thread per step at byte offset OFF (per stage)
template <int OFF, int BYTES>
struct Field {
  static constexpr int off = OFF, bytes = BYTES;
  static constexpr int U = Gran<BYTES>::U, N = Gran<BYTES>::N;
};

// Stage buffer of NT threads: `base` points at this stage's shared bytes.
template <int NT>
struct Stage {
  unsigned char* base;
  template <class F>
  __device__ __forceinline__ void fetch(const void* src) const {
    const unsigned char* s = static_cast<const unsigned char*>(src);
#pragma unroll
    for (int g = 0; g < F::N; ++g)
      cp_async<F::U>(base + F::off * NT + g * F::U * NT + threadIdx.x * F::U, s + g * F::U);
  }
  template <class F, typename S, int R, int C>
  __device__ __forceinline__ Mat<S, R, C> get() const {
    static_assert(R * C * (int)sizeof(S) == F::bytes, "field size");
    Mat<S, R, C> m;
    S* o = &m.a[0][0];
#pragma unroll
    for (int g = 0; g < F::N; ++g) {
      const unsigned char* p = base + F::off * NT + g * F::U * NT + threadIdx.x * F::U;
      if constexpr (F::U == 16) {
        const float4 v = *reinterpret_cast<const float4*>(p);
        const S* vs = reinterpret_cast<const S*>(&v);
#pragma unroll
        for (int j = 0; j < 16 / (int)sizeof(S); ++j) o[g * (16 / sizeof(S)) + j] = vs[j];
      } else if constexpr (F::U == 8) {
        const float2 v = *reinterpret_cast<const float2*>(p);
        const S* vs = reinterpret_cast<const S*>(&v);
#pragma unroll
        for (int j = 0; j < 8 / (int)sizeof(S); ++j) o[g * (8 / sizeof(S)) + j] = vs[j];
      } else {
        o[g] = *reinterpret_cast<const S*>(p);
      }
    }
    return m;
  }
};

// Per-step filter inputs (F, u, Q, H, d, R, y), byte offsets within a stage
// (multiplied by NT inside Stage)
template <typename S, int NX, int NY>
struct FilterIn {
  static constexpr int s = sizeof(S);
  using F = Field<0, NX * NX * s>;
  using u = Field<F::off + F::bytes, NX * s>;
  using Q = Field<u::off + u::bytes, NX * NX * s>;
  using H = Field<Q::off + Q::bytes, NY * NX * s>;
  using d = Field<H::off + H::bytes, NY * s>;
  using R = Field<d::off + d::bytes, NY * NY * s>;
  using y = Field<R::off + R::bytes, NY * s>;
  static constexpr int bytes = y::off + y::bytes;  // per thread per stage
};
// Per-step smoother inputs: filtered (x, P)_i and the transition (F, Q, u)_{i+1}
template <typename S, int NX>
struct SmootherIn {
  static constexpr int s = sizeof(S);
  using x = Field<0, NX * s>;
  using P = Field<x::off + x::bytes, NX * NX * s>;
  using F = Field<P::off + P::bytes, NX * NX * s>;
  using Q = Field<F::off + F::bytes, NX * NX * s>;
  using u = Field<Q::off + Q::bytes, NX * s>;
  static constexpr int bytes = u::off + u::bytes;
};

}  // namespace psk
