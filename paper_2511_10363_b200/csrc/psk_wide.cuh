// psk_wide.cuh -- the fast path for state dimensions the register-resident
// kernels do not cover (nx > 4 or ny > 4, up to the reference's kMaxDim = 16,
// mat.hpp:19): ONE WARP per chunk, matrices resident in shared memory.
//
// At nx = 16 a filtering element is 3 nx^2 + 2 nx = 800 scalars (6.4 KB in
// FP64) -- it cannot live in one thread's registers (hard part
// 1), so every matrix of a chunk lives in the warp's shared-memory slots and
// the 32 lanes cooperate on each operation: products (lanes over output
// entries), Cholesky / pivoted LU (sequential over columns, lanes over rows),
// triangular solves (lanes over right-hand-side columns).  Per step the work
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

// C[n x m] = (Z or 0) + sgn * op(A) op(B), op(X) = X or X^T; inner dim k.
// C must not alias A or B (it may alias Z: each entry reads Z first).
template <typename S>
__device__ __forceinline__ void gemm(WM<S> C, WM<S> A, bool tA, WM<S> B, bool tB, int n, int k,
                                     int m, const S* z = nullptr, int zld = 0, S sgn = S(1),
                                     bool sym = false) {
  for (int idx = lane_id(); idx < n * m; idx += 32) {
    const int r = idx / m, c = idx - (idx / m) * m;
    if (sym && c < r) continue;  // symmetric result: upper triangle, mirrored below
    S acc = z ? z[r * zld + c] : S(0);
    for (int q = 0; q < k; ++q) {
      const S a = tA ? A(q, r) : A(r, q);
      const S b = tB ? B(c, q) : B(q, c);
      acc = sfma(sgn * a, b, acc);
    }
    C(r, c) = acc;
    if (sym) C(c, r) = acc;
  }
  __syncwarp();
}
template <typename S>
__device__ __forceinline__ void copy(WM<S> D, WM<S> A, int n, int m) {
  for (int idx = lane_id(); idx < n * m; idx += 32) {
    const int r = idx / m, c = idx - (idx / m) * m;
    D(r, c) = A(r, c);
  }
  __syncwarp();
}
template <typename S>
__device__ __forceinline__ void fill(WM<S> D, int n, int m, S diag, S off) {
  for (int idx = lane_id(); idx < n * m; idx += 32) {
    const int r = idx / m, c = idx - (idx / m) * m;
    D(r, c) = r == c ? diag : off;
  }
  __syncwarp();
}
// coalesced load of a contiguous row-major r x c block from global
template <typename S>
__device__ __forceinline__ void gload(WM<S> D, const S* g, int n, int m) {
  for (int idx = lane_id(); idx < n * m; idx += 32) {
    const int r = idx / m, c = idx - (idx / m) * m;
    D(r, c) = g[idx];
  }
}
template <typename S>
__device__ __forceinline__ void gstore(S* g, WM<S> A, int n, int m) {
  for (int idx = lane_id(); idx < n * m; idx += 32) {
    const int r = idx / m, c = idx - (idx / m) * m;
    g[idx] = A(r, c);
  }
}

// Cholesky A = L L^T (mat.hpp:153-175): L lower (upper part unused), inv[j]
// = 1 / L(j,j).  Sequential over columns, lanes over the rows below.
template <typename S>
__device__ __forceinline__ void chol(WM<S> L, S* inv, WM<S> A, int n, unsigned& err) {
  for (int j = 0; j < n; ++j) {
    S d = A(j, j);
    for (int q = 0; q < j; ++q) d = sfma(-L(j, q), L(j, q), d);
    if (!(d > S(0))) err |= kErrNotPD;
    const S il = srsqrt(d);
    for (int i = j + lane_id(); i < n; i += 32) {
      if (i == j) {
        L(j, j) = d * il;
        inv[j] = il;
      } else {
        S acc = A(i, j);
        for (int q = 0; q < j; ++q) acc = sfma(-L(i, q), L(j, q), acc);
        L(i, j) = acc * il;
      }
    }
    __syncwarp();
  }
}
// X[n x m] = (L L^T)^-1 B; lanes over columns (X may alias B)
template <typename S>
__device__ __forceinline__ void chol_solve(WM<S> X, WM<S> L, const S* inv, WM<S> B, int n,
                                           int m) {
  for (int c = lane_id(); c < m; c += 32) {
    for (int i = 0; i < n; ++i) {
      S acc = B(i, c);
      for (int q = 0; q < i; ++q) acc = sfma(-L(i, q), X(q, c), acc);
      X(i, c) = acc * inv[i];
    }
    for (int i = n - 1; i >= 0; --i) {
      S acc = X(i, c);
      for (int q = i + 1; q < n; ++q) acc = sfma(-L(q, i), X(q, c), acc);
      X(i, c) = acc * inv[i];
    }
  }
  __syncwarp();
}

// LU with partial pivoting (mat.hpp:177-205): LU holds unit-lower L and U,
// inv[c] = 1 / U(c,c), piv[c] = row swapped into c at step c (first maximum
// of |a(r,c)|, as the reference).
template <typename S>
__device__ __forceinline__ void lu(WM<S> LU, S* inv, int* piv, int n, unsigned& err) {
  const int ln = lane_id();
  for (int c = 0; c < n; ++c) {
    // argmax over rows c..n-1 (lowest index on ties)
    S best = S(-1);
    int p = c;
    for (int r = c + ln; r < n; r += 32) {
      const S v = sabs(LU(r, c));
      if (v > best) { best = v; p = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const S ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int op = __shfl_xor_sync(0xffffffffu, p, o);
      if (ob > best || (ob == best && op < p)) { best = ob; p = op; }
    }
    if (ln == 0) piv[c] = p;
    if (best == S(0)) err |= kErrSingular;
    if (p != c)
      for (int j = ln; j < n; j += 32) {
        const S t = LU(c, j);
        LU(c, j) = LU(p, j);
        LU(p, j) = t;
      }
    __syncwarp();
    const S ip = srcp(LU(c, c));
    if (ln == 0) inv[c] = ip;
    for (int r = c + 1 + ln; r < n; r += 32) LU(r, c) *= ip;
    __syncwarp();
    const int w = n - c - 1;
    for (int idx = ln; idx < w * w; idx += 32) {
      const int r = c + 1 + idx / w, j = c + 1 + idx % w;
      LU(r, j) = sfma(-LU(r, c), LU(c, j), LU(r, j));
    }
    __syncwarp();
  }
}
// X = M^-1 B (trans = false) or M^-T B (trans = true); lanes over columns
template <typename S>
__device__ __forceinline__ void lu_solve(WM<S> X, WM<S> LU, const S* inv, const int* piv,
                                         WM<S> B, int n, int m, bool trans) {
  for (int c = lane_id(); c < m; c += 32) {
    if (!trans) {
      for (int i = 0; i < n; ++i) X(i, c) = B(i, c);
      for (int q = 0; q < n; ++q) {
        const int p = piv[q];
        if (p != q) {
          const S t = X(q, c);
          X(q, c) = X(p, c);
          X(p, c) = t;
        }
      }
      for (int i = 1; i < n; ++i) {
        S acc = X(i, c);
        for (int q = 0; q < i; ++q) acc = sfma(-LU(i, q), X(q, c), acc);
        X(i, c) = acc;
      }
      for (int i = n - 1; i >= 0; --i) {
        S acc = X(i, c);
        for (int q = i + 1; q < n; ++q) acc = sfma(-LU(i, q), X(q, c), acc);
        X(i, c) = acc * inv[i];
      }
    } else {
      for (int i = 0; i < n; ++i) {  // U^T z = b
        S acc = B(i, c);
        for (int q = 0; q < i; ++q) acc = sfma(-LU(q, i), X(q, c), acc);
        X(i, c) = acc * inv[i];
      }
      for (int i = n - 1; i >= 0; --i) {  // L^T w = z
        S acc = X(i, c);
        for (int q = i + 1; q < n; ++q) acc = sfma(-LU(q, i), X(q, c), acc);
        X(i, c) = acc;
      }
      for (int q = n - 1; q >= 0; --q) {  // undo the interchanges
        const int p = piv[q];
        if (p != q) {
          const S t = X(q, c);
          X(q, c) = X(p, c);
          X(p, c) = t;
        }
      }
    }
  }
  __syncwarp();
}

}  // namespace wide
}  // namespace psk
