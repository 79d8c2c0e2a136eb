// psk_wide.cuh -- the fast path for state dimensions the register-resident
// kernels do not cover (nx > 4 or ny > 4, up to the reference's kMaxDim = 16,
// mat.hpp:19): ONE WARP per chunk, matrices resident in shared memory.
//
// At nx = 16 a filtering element is 3 nx^2 + 2 nx = 800 scalars (6.4 KB in
// FP64) -- it cannot live in one thread's registers (hard part
// 1), so every matrix of a chunk lives in the warp's shared-memory slots and
// the 32 lanes cooperate on each operation: products (each lane a 2 x 4
// register tile of the output) and solves / inverses (Gauss-Jordan on an
// augmented block, each pivot step lane-parallel over the trailing block).  Per step the work
// is ~40 k flops (make_filter_element 40 676, Lemma-1 combine
// 88 624 at nx = 16), so the warp is busy; per-step model blocks are
// contiguous in the reference layout and a warp reads each with one
// coalesced sweep.  Dimensions are runtime (1..16); the formulation (chunked
// conditional Kalman reduce, scan, finish writing per-step smoothing
// elements) is the one of psk_fast.cuh.  Each lane writes through its own
// rows/columns; __syncwarp() separates the steps of every primitive.
#pragma once
#include <cuda_runtime.h>

#include "psk_common.cuh"
#include "psk_mat.cuh"

namespace psk {
namespace wide {

constexpr int kMaxN = 16;
constexpr int kLd = 17;                  // padded row stride: conflict-free columns
constexpr int kMat = kMaxN * kLd;        // scalars per matrix slot
constexpr int kVec = kMaxN;              // scalars per vector slot
constexpr int kWarps = 2;                // warps (chunks) per CTA

template <typename S>
struct WM {  // row-major matrix view in shared memory
  S* p;
  int ld;
  __device__ __forceinline__ S& operator()(int r, int c) const { return p[r * ld + c]; }
};
template <typename S>
__device__ __forceinline__ WM<S> mat(S* p) { return WM<S>{p, kLd}; }
template <typename S>
__device__ __forceinline__ WM<S> vec(S* p) { return WM<S>{p, 1}; }

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Element loops without integer division (runtime divisors cost ~20
// instructions each and dominated the first version's instruction mix,
// profiles/r01_v6): for m <= 16 lane l covers column l & 15 of rows
// l >> 4, l >> 4 + 2, ...; wider blocks go row by row, lanes over columns.
template <class Fn>
__device__ __forceinline__ void for_each(int n, int m, Fn&& fn) {
  const int ln = lane_id();
  if (m <= 16) {
    const int c = ln & 15;
    if (c < m)
      for (int r = ln >> 4; r < n; r += 2) fn(r, c);
  } else {
    for (int r = 0; r < n; ++r)
      for (int c = ln; c < m; c += 32) fn(r, c);
  }
}

// C[n x m] = (Z or 0) + sgn * op(A) op(B), op(X) = X or X^T (TA, TB); inner
// dim k.  Register-blocked: each lane owns a 2 x 4 tile of C (8 independent
// accumulators: a one-output-per-lane dot product is a chain of dependent
// FMAs), operands walked by pointer increments; a matrix-vector product uses
// lanes over rows with 4 partial sums.  `sym`: the result is symmetric --
// tiles below the diagonal are skipped and the upper triangle is mirrored.
// C must not alias A or B (it may alias Z entry-wise).
template <bool TA, bool TB, typename S>
__device__ __forceinline__ void gemm(WM<S> C, WM<S> A, WM<S> B, int n, int k, int m,
                                     const S* z = nullptr, int zld = 0, S sgn = S(1),
                                     bool sym = false) {
  const int as = TA ? A.ld : 1;   // step of op(A)(r, q) in q
  const int bs = TB ? 1 : B.ld;   // step of op(B)(q, c) in q
  if (m == 1) {
    for (int r = lane_id(); r < n; r += 32) {
      const S* pa = TA ? &A(0, r) : &A(r, 0);
      const S* pb = &B(0, 0);
      S acc[4] = {S(0), S(0), S(0), S(0)};
      int q = 0;
      for (; q + 4 <= k; q += 4) {
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = sfma(pa[(q + j) * as], pb[(q + j) * bs], acc[j]);
      }
      for (; q < k; ++q) acc[0] = sfma(pa[q * as], pb[q * bs], acc[0]);
      const S sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
      C(r, 0) = sfma(sgn, sum, z ? z[r * zld] : S(0));
    }
    __syncwarp();
    return;
  }
  const int tr = (n + 1) >> 1, tc = (m + 3) >> 2;
  for (int t = lane_id(); t < tr * tc; t += 32) {
    const int r0 = (t / tc) * 2, c0 = (t - (t / tc) * tc) * 4;
    if (sym && c0 + 3 < r0) continue;  // entirely below the diagonal
    const int r1 = min(r0 + 1, n - 1);
    const S* pa0 = TA ? &A(0, r0) : &A(r0, 0);
    const S* pa1 = TA ? &A(0, r1) : &A(r1, 0);
    const S* pb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cj = min(c0 + j, m - 1);
      pb[j] = TB ? &B(cj, 0) : &B(0, cj);
    }
    S acc[2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = S(0);
#pragma unroll 4
    for (int q = 0; q < k; ++q) {
      const S a0 = pa0[q * as], a1 = pa1[q * as];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const S b = pb[j][q * bs];
        acc[0][j] = sfma(a0, b, acc[0][j]);
        acc[1][j] = sfma(a1, b, acc[1][j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + i, c = c0 + j;
        if (r < n && c < m && (!sym || c >= r))
          C(r, c) = sfma(sgn, acc[i][j], z ? z[r * zld + c] : S(0));
      }
  }
  __syncwarp();
  if (sym) {
    for_each(n, n, [&](int r, int c) {
      if (c < r) C(r, c) = C(c, r);
    });
    __syncwarp();
  }
}
template <typename S>
__device__ __forceinline__ void copy(WM<S> D, WM<S> A, int n, int m) {
  for_each(n, m, [&](int r, int c) { D(r, c) = A(r, c); });
  __syncwarp();
}
template <typename S>
__device__ __forceinline__ void fill(WM<S> D, int n, int m, S diag, S off) {
  for_each(n, m, [&](int r, int c) { D(r, c) = r == c ? diag : off; });
  __syncwarp();
}
// coalesced load / store of a contiguous row-major n x m block in global
template <typename S>
__device__ __forceinline__ void gload(WM<S> D, const S* g, int n, int m) {
  for_each(n, m, [&](int r, int c) { D(r, c) = g[r * m + c]; });
}
template <typename S>
__device__ __forceinline__ void gstore(S* g, WM<S> A, int n, int m) {
  for_each(n, m, [&](int r, int c) { g[r * m + c] = A(r, c); });
}

// Gauss-Jordan elimination on the augmented n x w matrix X = [A | B]
// (n <= 16, w <= 64): the left block is reduced to I and the same row
// operations turn the right block into A^-1 B.  Column-oriented and
// register-resident: lane l holds columns l and l + 32 in registers, every
// pivot step broadcasts the pivot column with shuffles and each lane updates
// its columns with independent FMAs (the shared-memory formulation spent
// half of k_wide_finish in load/store chains of this elimination,
// profiles/r01_v6).  The pivot loop is unrolled so every register index is
// static.  pivot = false: A symmetric positive definite, no row exchanges
// (elimination on an SPD matrix is stable; a non-positive pivot raises
// kErrNotPD as the reference's Cholesky does, mat.hpp:165); pivot = true:
// partial pivoting on the first maximum |a(r, p)| (mat.hpp:180-205), a zero
// pivot raises kErrSingular.
template <typename S>
__device__ __forceinline__ void gauss_jordan(WM<S> X, int n, int w, bool pivot, unsigned& err) {
  const int ln = lane_id();
  const bool has0 = ln < w, has1 = ln + 32 < w;
  S x0[kMaxN], x1[kMaxN];
#pragma unroll
  for (int i = 0; i < kMaxN; ++i) {
    x0[i] = (i < n && has0) ? X(i, ln) : S(0);
    x1[i] = (i < n && has1) ? X(i, ln + 32) : S(0);
  }
#pragma unroll
  for (int p = 0; p < kMaxN; ++p) {
    if (p >= n) break;
    if (pivot) {
      // lane p holds the pivot column: first maximum of |x(i, p)|, i >= p
      S best = S(-1);
      int pr = p;
#pragma unroll
      for (int i = p; i < kMaxN; ++i)
        if (i < n && sabs(x0[i]) > best) { best = sabs(x0[i]); pr = i; }
      pr = __shfl_sync(0xffffffffu, pr, p);
      best = __shfl_sync(0xffffffffu, best, p);
      if (best == S(0)) err |= kErrSingular;
      if (pr != p) {  // warp-uniform: swap rows p and pr in every column
        S a0 = x0[p], a1 = x1[p];
#pragma unroll
        for (int i = p + 1; i < kMaxN; ++i)
          if (i == pr) {
            x0[p] = x0[i];
            x1[p] = x1[i];
            x0[i] = a0;
            x1[i] = a1;
          }
      }
    }
    const S d = __shfl_sync(0xffffffffu, x0[p], p);
    if (!pivot && !(d > S(0))) err |= kErrNotPD;
    const S ip = srcp(d);
    const S r0 = x0[p] * ip, r1 = x1[p] * ip;  // scaled pivot row (my columns)
#pragma unroll
    for (int i = 0; i < kMaxN; ++i) {
      if (i >= n) break;
      const S f = __shfl_sync(0xffffffffu, x0[i], p);  // pivot column entry
      if (i != p) {
        x0[i] = sfma(-f, r0, x0[i]);
        x1[i] = sfma(-f, r1, x1[i]);
      }
    }
    x0[p] = r0;
    x1[p] = r1;
  }
#pragma unroll
  for (int i = 0; i < kMaxN; ++i) {
    if (i >= n) break;
    if (has0) X(i, ln) = x0[i];
    if (has1) X(i, ln + 32) = x1[i];
  }
  __syncwarp();
}

}  // namespace wide
}  // namespace psk
