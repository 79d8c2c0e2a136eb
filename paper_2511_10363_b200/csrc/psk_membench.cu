// psk_membench.cu -- memory-pattern microbenchmark of the chunk walk
// (measurement tool, built into libpsk_tools.so; not part of the product).
//
// The fast path's per-step kernels walk one chunk of L consecutive steps per
// thread over the reference's per-step model layout (7 arrays of per-step
// blocks, 416 B per step at nx=4, ny=2, f64).  This isolates the memory side
// of that walk from its arithmetic: every variant reads the same 7 GB and
// only sums what it read.
//   stream   grid-stride contiguous 16-byte loads (the HBM read ceiling)
//   direct   per-thread walk, vector loads straight from global
//   coop     per-thread walk fed by the warp-cooperative cp.async stage
//            (psk_stage.cuh), double-buffered
// Occupancy is set with a dynamic shared-memory reservation (`ctas` CTAs of
// 128 threads per SM) so the variants can be compared at the 8 warps/SM of
// the 255-register FP64 kernels.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "psk_stage.cuh"

// ---- LDGSTS (cp.async) staging variants measured against TMA below; the
// product kernels stage with TMA (psk_stage.cuh) because of these numbers.
namespace psk {
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

// A field of BYTES bytes per thread per step, starting at byte OFF of a
// stage of NT threads.
template <int NT, int OFF, int BYTES>
struct Field {
  static constexpr int U = BYTES % 16 == 0 ? 16 : (BYTES % 8 == 0 ? 8 : 4);
  static constexpr int N = BYTES / U;
  static constexpr int row = NT * U + 16;  // bytes per granule row (padded)
  static constexpr int off = OFF, bytes = BYTES;
  static constexpr int end = OFF + N * row;
};

// Warp-cooperative fetch of one field for the warp's 32 chunks at one walk
// position.  The block of warp-thread tl starts at base + k(tl) * stride
// scalars with k(tl) = (cw0 + tl) * L + j.  When N divides 32, lane l always
// moves granule g = l % N of warp-threads tl = l / N + (32 / N) i, so its
// source pointers form an arithmetic progression (no per-granule index
// math); `full` says all 32 chunks of the warp have step j.
template <class F, typename S>
__device__ __forceinline__ void coop_fetch(unsigned char* stage, const S* base,
                                           long long stride, long long cw0, long long L,
                                           long long j, long long nchunks, long long t,
                                           bool full, int warp_t0, int lane) {
  constexpr int N = F::N, U = F::U;
  if constexpr (32 % N == 0) {
    constexpr int TS = 32 / N;  // warp-threads per request
    const int g = lane % N, tl0 = lane / N;
    const long long k0 = (cw0 + tl0) * L + j;
    const unsigned char* p =
        reinterpret_cast<const unsigned char*>(base + k0 * stride) + g * U;
    const long long di = (long long)TS * L * stride * (long long)sizeof(S);
    unsigned char* d = stage + F::off + g * F::row + (warp_t0 + tl0) * U;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (full || (cw0 + tl0 + TS * i < nchunks && k0 + (long long)TS * i * L < t))
        cp_async<U>(d + TS * i * U, p + i * di);
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int idx = lane + 32 * i;
      const int tl = idx / N, g = idx % N;
      const long long c = cw0 + tl;
      const long long k = c * L + j;
      if (c < nchunks && k < t)
        cp_async<U>(stage + F::off + g * F::row + (warp_t0 + tl) * U,
                    reinterpret_cast<const unsigned char*>(base + k * stride) + g * U);
    }
  }
}

// This thread's block of a field as a matrix (row-major R x C).
template <class F, typename S, int R, int C>
__device__ __forceinline__ Mat<S, R, C> stage_get(const unsigned char* stage, int t) {
  static_assert(R * C * (int)sizeof(S) == F::bytes, "field size");
  Mat<S, R, C> m;
  S* o = &m.a[0][0];
#pragma unroll
  for (int g = 0; g < F::N; ++g) {
    const unsigned char* p = stage + F::off + g * F::row + t * F::U;
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

// Per-step filter inputs (F, u, Q, H, d, R, y) of a stage of NT threads
template <typename S, int NX, int NY, int NT>
struct FilterIn {
  static constexpr int s = sizeof(S);
  using F = Field<NT, 0, NX * NX * s>;
  using u = Field<NT, F::end, NX * s>;
  using Q = Field<NT, u::end, NX * NX * s>;
  using H = Field<NT, Q::end, NY * NX * s>;
  using d = Field<NT, H::end, NY * s>;
  using R = Field<NT, d::end, NY * NY * s>;
  using y = Field<NT, R::end, NY * s>;
  static constexpr int bytes = (y::end + 127) / 128 * 128;  // one stage
};

}  // namespace psk

namespace {

using psk::FilterIn;
constexpr int NT = 128;
using In = FilterIn<double, 4, 2, NT>;

struct Model {
  const double *f, *u, *q, *h, *d, *r, *y;
  long long t;
};

__global__ void __launch_bounds__(256) k_stream(const float4* const* arr, const long long* n,
                                                int narr, double* out) {
  double acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int a = 0; a < narr; ++a) {
    const float4* p = arr[a];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n[a]; i += stride) {
      const float4 v = __ldcs(p + i);
      acc += v.x + v.y + v.z + v.w;
    }
  }
  if (acc == -1.2345) out[0] = acc;
}

template <int R>
__device__ __forceinline__ double sum_blk(const double* p) {
  double s = 0;
  const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int i = 0; i < R / 2; ++i) {
    const float4 v = __ldg(q + i);
    const double* d = reinterpret_cast<const double*>(&v);
    s += d[0] + d[1];
  }
  return s;
}

__global__ void __launch_bounds__(NT) k_direct(Model m, long long L, double* out) {
  extern __shared__ unsigned char pad[];
  const long long c = (long long)blockIdx.x * NT + threadIdx.x;
  const long long k0 = c * L, k1 = min(k0 + L, m.t);
  double acc = 0;
  for (long long k = k0; k < k1; ++k) {
    acc += sum_blk<16>(m.f + k * 16) + sum_blk<4>(m.u + k * 4) + sum_blk<16>(m.q + k * 16) +
           sum_blk<8>(m.h + k * 8) + sum_blk<2>(m.d + k * 2) + sum_blk<4>(m.r + k * 4) +
           sum_blk<2>(m.y + k * 2);
  }
  if (acc == -1.2345) out[0] = acc + pad[0];
}

template <class F>
__device__ __forceinline__ double sum_stage(const unsigned char* st, int t) {
  double s = 0;
#pragma unroll
  for (int g = 0; g < F::N; ++g) {
    const float4 v = *reinterpret_cast<const float4*>(st + F::off + g * F::row + t * 16);
    const double* d = reinterpret_cast<const double*>(&v);
    s += d[0] + d[1];
  }
  return s;
}

__device__ __forceinline__ void fetch(unsigned char* st, const Model& m, long long L,
                                      long long nch, long long cw0, long long j, bool full,
                                      int wt0, int lane) {
  psk::coop_fetch<In::F>(st, m.f, 16, cw0, L, j, nch, m.t, full, wt0, lane);
  psk::coop_fetch<In::u>(st, m.u, 4, cw0, L, j, nch, m.t, full, wt0, lane);
  psk::coop_fetch<In::Q>(st, m.q, 16, cw0, L, j, nch, m.t, full, wt0, lane);
  psk::coop_fetch<In::H>(st, m.h, 8, cw0, L, j, nch, m.t, full, wt0, lane);
  psk::coop_fetch<In::d>(st, m.d, 2, cw0, L, j, nch, m.t, full, wt0, lane);
  psk::coop_fetch<In::R>(st, m.r, 4, cw0, L, j, nch, m.t, full, wt0, lane);
  psk::coop_fetch<In::y>(st, m.y, 2, cw0, L, j, nch, m.t, full, wt0, lane);
}

template <int DEPTH>
__global__ void __launch_bounds__(NT) k_coop(Model m, long long L, long long nch, double* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, wt0 = threadIdx.x & ~31;
  const long long cw0 = (long long)blockIdx.x * NT + wt0;
  if (cw0 >= nch) return;
  const long long jn = min(L, m.t - cw0 * L);
  const bool full = (cw0 + 32) * L <= m.t;
  const long long c = cw0 + lane;
  const long long k0 = c * L, k1 = min(k0 + L, m.t);
  double acc = 0;
#pragma unroll
  for (int s = 0; s < DEPTH - 1; ++s) {
    if (s < jn) fetch(sm + s * In::bytes, m, L, nch, cw0, s, full, wt0, lane);
    psk::cp_async_commit();
  }
  for (long long j = 0; j < jn; ++j) {
    const long long jf = j + DEPTH - 1;
    if (jf < jn) fetch(sm + (jf % DEPTH) * In::bytes, m, L, nch, cw0, jf, full, wt0, lane);
    psk::cp_async_commit();
    psk::cp_async_wait<DEPTH - 1>();
    __syncwarp();
    if (k0 + j < k1) {
      const unsigned char* st = sm + (j % DEPTH) * In::bytes;
      const int t = threadIdx.x;
      acc += sum_stage<In::F>(st, t) + sum_stage<In::u>(st, t) + sum_stage<In::Q>(st, t) +
             sum_stage<In::H>(st, t) + sum_stage<In::d>(st, t) + sum_stage<In::R>(st, t) +
             sum_stage<In::y>(st, t);
    }
    __syncwarp();
  }
  if (acc == -1.2345) out[0] = acc;
}

// ---- per-thread TMA bulk copies (cp.async.bulk), one mbarrier per thread
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(psk::smem_u32(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   psk::smem_u32(b)),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(psk::smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          psk::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(psk::smem_u32(b))
      : "memory");
}
constexpr int kThr = 432;  // per-thread stage bytes (416 + 16 pad: conflict-free)

__device__ __forceinline__ void bulk_fetch(unsigned char* slot, uint64_t* b, const Model& m,
                                           long long k) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect(b, 416);
  bulk_g2s(slot, m.f + k * 16, 128, b);
  bulk_g2s(slot + 128, m.u + k * 4, 32, b);
  bulk_g2s(slot + 160, m.q + k * 16, 128, b);
  bulk_g2s(slot + 288, m.h + k * 8, 64, b);
  bulk_g2s(slot + 352, m.d + k * 2, 16, b);
  bulk_g2s(slot + 368, m.r + k * 4, 32, b);
  bulk_g2s(slot + 400, m.y + k * 2, 16, b);
}

template <int DEPTH>
__global__ void __launch_bounds__(NT) k_bulk(Model m, long long L, double* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + DEPTH * NT * kThr);
  const int t = threadIdx.x;
  const long long c = (long long)blockIdx.x * NT + t;
  const long long k0 = c * L, k1 = min(k0 + L, m.t);
  for (int s = 0; s < DEPTH; ++s) mbar_init(&bars[s * NT + t], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  double acc = 0;
  for (int s = 0; s < DEPTH - 1; ++s)
    if (k0 + s < k1) bulk_fetch(sm + (s * NT + t) * kThr, &bars[s * NT + t], m, k0 + s);
  for (long long k = k0; k < k1; ++k) {
    const long long j = k - k0;
    const long long jf = j + DEPTH - 1;
    if (k0 + jf < k1) {
      const int sf = (int)(jf % DEPTH);
      bulk_fetch(sm + (sf * NT + t) * kThr, &bars[sf * NT + t], m, k0 + jf);
    }
    const int s = (int)(j % DEPTH);
    mbar_wait(&bars[s * NT + t], (unsigned)((j / DEPTH) & 1));
    const float4* q = reinterpret_cast<const float4*>(sm + (s * NT + t) * kThr);
#pragma unroll
    for (int i = 0; i < 26; ++i) {
      const float4 v = q[i];
      const double* d = reinterpret_cast<const double*>(&v);
      acc += d[0] + d[1];
    }
  }
  if (acc == -1.2345) out[0] = acc;
}

// persistent CTAs walking tiles of NT consecutive steps (L = 1 access
// pattern without per-CTA launch cost): tile b+grid is in flight while tile
// b is summed.  `span` > 1 spreads the tile: thread t takes step b*NT*span +
// t*span (so consecutive lanes are span steps apart, the chunked pattern).
template <int DEPTH>
__global__ void __launch_bounds__(NT) k_coop_persist(Model m, long long span, double* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, wt0 = threadIdx.x & ~31;
  const long long ntile = (m.t / span + NT - 1) / NT;
  double acc = 0;
  // tile b of "chunks" of length span: fetch position j = (b * NT) ... we
  // emulate chunk walks of length span with all 32 lanes at one walk position
  const long long nch = (m.t + span - 1) / span;
  long long it = 0;
  for (long long b = blockIdx.x; b < ntile * span; b += gridDim.x, ++it) {
    (void)b;
  }
  const long long nit = it;  // tiles (x walk positions) of this CTA
  auto pos = [&](long long i, long long& cw0, long long& j) {
    const long long q = blockIdx.x + i * gridDim.x;  // global work item
    const long long tile = q / span;
    j = q % span;
    cw0 = tile * NT + wt0;
  };
  for (int s = 0; s < DEPTH - 1; ++s) {
    if (s < nit) {
      long long cw0, j;
      pos(s, cw0, j);
      fetch(sm + s * In::bytes, m, span, nch, cw0, j, (cw0 + 32) * span <= m.t, wt0, lane);
    }
    psk::cp_async_commit();
  }
  for (long long i = 0; i < nit; ++i) {
    const long long i_f = i + DEPTH - 1;
    if (i_f < nit) {
      long long cw0, j;
      pos(i_f, cw0, j);
      fetch(sm + (i_f % DEPTH) * In::bytes, m, span, nch, cw0, j, (cw0 + 32) * span <= m.t,
            wt0, lane);
    }
    psk::cp_async_commit();
    psk::cp_async_wait<DEPTH - 1>();
    __syncwarp();
    const unsigned char* st = sm + (i % DEPTH) * In::bytes;
    const int t = threadIdx.x;
    acc += sum_stage<In::F>(st, t) + sum_stage<In::u>(st, t) + sum_stage<In::Q>(st, t) +
           sum_stage<In::H>(st, t) + sum_stage<In::d>(st, t) + sum_stage<In::R>(st, t) +
           sum_stage<In::y>(st, t);
    __syncwarp();
  }
  if (acc == -1.2345) out[0] = acc;
}

// ---- TMA tensor maps: each field viewed as [blk, L, nchunks] (3-D), one
// box {blk, 1, NT} per field per step = the step of all NT chunks of a CTA;
// the box rows are swizzled so per-thread 16-byte reads are conflict-free.
struct TMaps {
  CUtensorMap m[7];
};
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                     uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(psk::smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(psk::smem_u32(b))
      : "memory");
}
__host__ __device__ constexpr int row_bytes(int f) {
  return f == 0 || f == 2 ? 128 : (f == 3 ? 64 : (f == 1 || f == 5 ? 32 : 16));
}
__host__ __device__ constexpr int box_off(int f) {
  int o = 0;
  for (int i = 0; i < f; ++i) o += (row_bytes(i) * NT + 1023) / 1024 * 1024;
  return o;
}
constexpr int kTmaStage = box_off(7);
// byte offset of 16-byte chunk c of row r in a box of R-byte rows (swizzle
// 128B / 64B / 32B for R = 128 / 64 / 32, none for 16)
__device__ __forceinline__ int swz(int r, int c, int R) {
  const int a = r * R + c * 16;
  const int m = R == 128 ? 7 : (R == 64 ? 3 : (R == 32 ? 1 : 0));
  return a ^ (((a >> 7) & m) << 4);
}
template <int DEPTH>
__global__ void __launch_bounds__(NT) k_tma(const __grid_constant__ TMaps maps, long long L,
                                            double* out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + DEPTH * kTmaStage);
  const int t = threadIdx.x;
  const int c2 = blockIdx.x * NT;
  if (t == 0) {
    for (int s = 0; s < DEPTH; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int s, int j) {
    mbar_expect(&bars[s], NT * 416);
    for (int f = 0; f < 7; ++f) tma3(sm + s * kTmaStage + box_off(f), &maps.m[f], 0, j, c2, &bars[s]);
  };
  if (t == 0)
    for (int s = 0; s < DEPTH - 1 && s < L; ++s) issue(s, s);
  double acc = 0;
  for (int j = 0; j < L; ++j) {
    if (t == 0 && j + DEPTH - 1 < L) issue((j + DEPTH - 1) % DEPTH, j + DEPTH - 1);
    const int s = j % DEPTH;
    mbar_wait(&bars[s], (unsigned)((j / DEPTH) & 1));
    const unsigned char* st = sm + s * kTmaStage;
#pragma unroll
    for (int f = 0; f < 7; ++f) {
      const int R = row_bytes(f);
#pragma unroll
      for (int c = 0; c < R / 16; ++c) {
        const float4 v = *reinterpret_cast<const float4*>(st + box_off(f) + swz(t, c, R));
        const double* d = reinterpret_cast<const double*>(&v);
        acc += d[0] + d[1];
      }
    }
    __syncthreads();  // stage s is refilled next iteration
  }
  if (acc == -1.2345) out[0] = acc;
}

float time_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

}  // namespace

// Runs every variant on device `device` with T steps and prints one JSON line
// per variant: {"variant", "L", "ctas_per_sm", "depth", "ms", "GBps"}.
extern "C" int psk_membench(int device, long long T) {
  cudaSetDevice(device);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, device);
  const int blk[7] = {16, 4, 16, 8, 2, 4, 2};
  double* a[7];
  size_t total = 0;
  for (int i = 0; i < 7; ++i) {
    if (cudaMalloc(&a[i], sizeof(double) * blk[i] * T) != cudaSuccess) return 1;
    cudaMemset(a[i], 0, sizeof(double) * blk[i] * T);
    total += sizeof(double) * blk[i] * T;
  }
  Model m{a[0], a[1], a[2], a[3], a[4], a[5], a[6], T};
  double* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t smem_sm = p.sharedMemPerMultiprocessor;
  auto report = [&](const char* v, long long L, int ctas, int depth, float ms) {
    printf("{\"variant\": \"%s\", \"L\": %lld, \"ctas_per_sm\": %d, \"depth\": %d, "
           "\"ms\": %.4f, \"GBps\": %.1f}\n",
           v, L, ctas, depth, ms, total / (ms * 1e-3) / 1e9);
    fflush(stdout);
  };
  // stream
  {
    const float4** d_arr;
    long long* d_n;
    cudaMalloc(&d_arr, sizeof(void*) * 7);
    cudaMalloc(&d_n, sizeof(long long) * 7);
    const float4* h_arr[7];
    long long h_n[7];
    for (int i = 0; i < 7; ++i) {
      h_arr[i] = reinterpret_cast<const float4*>(a[i]);
      h_n[i] = (long long)blk[i] * T / 2;
    }
    cudaMemcpy(d_arr, h_arr, sizeof(h_arr), cudaMemcpyHostToDevice);
    cudaMemcpy(d_n, h_n, sizeof(h_n), cudaMemcpyHostToDevice);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0);
      k_stream<<<p.multiProcessorCount * 8, 256>>>(d_arr, d_n, 7, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      best = fminf(best, time_ms(e0, e1));
    }
    report("stream", 0, 8, 0, best);
  }
  for (long long span : {1LL, 4LL, 16LL, 64LL}) {
    for (int depth : {2, 3}) {
      const size_t sm = (size_t)depth * In::bytes;
      const int ctas = (int)(smem_sm / (sm + 1024));
      auto kern = depth == 2 ? k_coop_persist<2> : k_coop_persist<3>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        kern<<<p.multiProcessorCount * ctas, NT, sm>>>(m, span, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        best = fminf(best, time_ms(e0, e1));
      }
      report("coop_persist", span, ctas, depth, best);
    }
  }
  {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc),
                            cudaEnableDefault, &q);
    for (long long L : {16LL, 64LL, 256LL}) {
      const long long nch = T / L;
      TMaps maps;
      bool ok = enc != nullptr;
      for (int f = 0; f < 7 && ok; ++f) {
        const int R = row_bytes(f);
        cuuint64_t dims[3] = {(cuuint64_t)(R / 8), (cuuint64_t)L, (cuuint64_t)nch};
        cuuint64_t strides[2] = {(cuuint64_t)R, (cuuint64_t)R * L};
        cuuint32_t box[3] = {(cuuint32_t)(R / 8), 1, NT};
        cuuint32_t es[3] = {1, 1, 1};
        const CUtensorMapSwizzle sw = R == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                     : R == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                     : R == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                               : CU_TENSOR_MAP_SWIZZLE_NONE;
        CUresult r = enc(&maps.m[f], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a[f], dims, strides, box,
                         es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          printf("{\"error\": \"tensor map %d: %d\"}\n", f, (int)r);
          ok = false;
        }
      }
      if (!ok) break;
      for (int depth : {2, 3}) {
        const size_t sm = (size_t)depth * kTmaStage + 1024 + 64;
        const int ctas = (int)(smem_sm / (sm + 1024));
        auto kern = depth == 2 ? k_tma<2> : k_tma<3>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
          cudaEventRecord(e0);
          kern<<<(unsigned)(nch / NT), NT, sm>>>(maps, L, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          best = fminf(best, time_ms(e0, e1));
        }
        report("tma", L, ctas, depth, best);
      }
    }
  }
  const long long Ls[1] = {64};
  const int ctas_list[3] = {2, 4, 8};
  for (long long L : Ls) {
    const long long nch = (T + L - 1) / L;
    const int grid = (int)((nch + NT - 1) / NT);
    for (int ctas : ctas_list) {
      // direct: reserve shared memory so that only `ctas` CTAs fit per SM
      const size_t pad = smem_sm / ctas - 1024 - 16;
      cudaFuncSetAttribute(k_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pad);
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        k_direct<<<grid, NT, pad>>>(m, L, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        best = fminf(best, time_ms(e0, e1));
      }
      report("direct", L, ctas, 0, best);
    }
    for (int depth : {2, 3}) {
      const size_t sm = (size_t)depth * In::bytes;
      const int ctas = (int)(smem_sm / (sm + 1024));
      auto kern = depth == 2 ? k_coop<2> : k_coop<3>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        kern<<<grid, NT, sm>>>(m, L, nch, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        best = fminf(best, time_ms(e0, e1));
      }
      report("coop", L, ctas, depth, best);
    }
    for (int depth : {2, 3, 4}) {
      const size_t sm = (size_t)depth * NT * kThr + depth * NT * 8;
      if (sm > 227 * 1024) continue;
      const int ctas = (int)(smem_sm / (sm + 1024));
      auto kern = depth == 2 ? k_bulk<2> : (depth == 3 ? k_bulk<3> : k_bulk<4>);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        kern<<<grid, NT, sm>>>(m, L, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        best = fminf(best, time_ms(e0, e1));
      }
      report("bulk", L, ctas, depth, best);
    }
  }
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
    return 2;
  }
  for (int i = 0; i < 7; ++i) cudaFree(a[i]);
  cudaFree(out);
  return 0;
}
