// psk_peak.cu -- FP64 / FP32 FMA-pipe peak microbenchmark (measurement tool
// for the roofline denominators that MEASURED_PEAKS.json does not carry; not
// part of the C-ABI product).  Built into libpsk_tools.so.
#include <cuda_runtime.h>

#include <cstdio>

namespace {

template <typename T>
__global__ void __launch_bounds__(256) k_fma(T* out, int iters, T a, T b) {
  // 8 independent chains per thread keep the FMA pipe full
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4,
    x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  T s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == T(-12345)) out[0] = s;  // keep the chains live
}

template <typename T>
int run(int device, double* tflops, double* ms_out) {
  cudaSetDevice(device);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, device);
  T* out;
  cudaMalloc(&out, sizeof(T));
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_fma<T><<<blocks, threads>>>(out, 64, T(0.999999), T(1e-7));  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_fma<T><<<blocks, threads>>>(out, iters, T(0.999999), T(1e-7));
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return 5;
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  *ms_out = best;
  return 0;
}

// FP64 tensor-core MMA (mma.sync m8n8k4 f64, DMMA): 8 independent 8x8
// accumulators per warp, operands in registers -- the ceiling a register-
// fragment formulation of the nx = 16 products could reach
__global__ void __launch_bounds__(256) k_dmma(double* out, int iters, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-9, b = b0;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
            : "+d"(c[i][0]), "+d"(c[i][1])
            : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == -12345.0) out[0] = s;
}

int run_dmma(int device, double* tflops, double* ms_out) {
  cudaSetDevice(device);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, device);
  double* out;
  cudaMalloc(&out, sizeof(double));
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 2048;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_dmma<<<blocks, threads>>>(out, 16, 1e-3, 1e-3);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_dmma<<<blocks, threads>>>(out, iters, 1e-3, 1e-3);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return 5;
  // one m8n8k4 = 8 * 8 * 4 FMA = 512 flops per warp
  const double flops = 512.0 * 32 * (double)iters * blocks * (threads / 32);
  *tflops = flops / (best * 1e-3) / 1e12;
  *ms_out = best;
  return 0;
}

}  // namespace

extern "C" int psk_peak_dmma(int device, double* tflops, double* ms) {
  return run_dmma(device, tflops, ms);
}

extern "C" int psk_peak_fma(int device, int f64, double* tflops, double* ms) {
  return f64 ? run<double>(device, tflops, ms) : run<float>(device, tflops, ms);
}

// ---- device reciprocal checks (tests/test_gpu_numerics.py) -----------------
// The fast path's branch-free srcp / srsqrt (psk_mat.cuh) over host arrays, so
// a test can hold them to the IEEE quotient the reference computes, including
// subnormal and huge arguments.
#include "psk_mat.cuh"

namespace {
template <typename T>
__global__ void k_rcp(const T* x, T* r, T* q, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    r[i] = psk::srcp(x[i]);
    q[i] = psk::srsqrt(x[i]);
  }
}
template <typename T>
int rcp_run(const void* x, void* r, void* q, int n) {
  T *dx, *dr, *dq;
  const size_t b = sizeof(T) * (size_t)(n > 0 ? n : 1);
  if (cudaMalloc(&dx, b) || cudaMalloc(&dr, b) || cudaMalloc(&dq, b)) return 8;
  cudaMemcpy(dx, x, sizeof(T) * n, cudaMemcpyHostToDevice);
  k_rcp<T><<<(n + 127) / 128 > 0 ? (n + 127) / 128 : 1, 128>>>(dx, dr, dq, n);
  cudaMemcpy(r, dr, sizeof(T) * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(q, dq, sizeof(T) * n, cudaMemcpyDeviceToHost);
  cudaFree(dx);
  cudaFree(dr);
  cudaFree(dq);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
}  // namespace

extern "C" int psk_tool_rcp(int f64, const void* x, void* rcp, void* rsqrt, int n) {
  return f64 ? rcp_run<double>(x, rcp, rsqrt, n) : rcp_run<float>(x, rcp, rsqrt, n);
}
