// psk_mat.cuh -- register-resident small-matrix kernels for the fast path.
//
// Replaces the reference's mat.hpp routines (mat.hpp:101-269) on the device:
// all dimensions are compile-time, every loop is fully unrolled, so matrices
// live in registers and no local memory is touched.  Arithmetic uses FMA and
// reciprocal pivots; row pivoting is done with predicated swaps (no dynamic
// register indexing).  These are NOT bit-compatible with the reference
// (psk_exact.cu is); parity is within the tolerances stated in DESIGN.md.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "psk_common.cuh"

namespace psk {

template <typename S, int R, int C>
struct Mat {
  S a[R][C];
  __device__ __forceinline__ S& operator()(int i, int j) { return a[i][j]; }
  __device__ __forceinline__ const S& operator()(int i, int j) const {
    return a[i][j];
  }
};
template <typename S, int N>
using Vec = Mat<S, N, 1>;


template <typename S>
__device__ __forceinline__ S sabs(S x) {
  return x < S(0) ? -x : x;
}
// Branch-free reciprocal and reciprocal square root: the MUFU approximation
// refined by Newton steps (quadratic convergence; two steps take the FP64
// seed below 1 ulp).  IEEE `1.0 / x` and `sqrt(x)` compile to a fast path
// plus a slow-path branch each, which splits every per-step body into many
// basic blocks and stops the scheduler from overlapping the independent
// filter / smoother-element / fold dependency chains (profiles/r01_v2).
// correctly rounded square root (exact mode: bitwise with the reference)
__device__ __forceinline__ double ssqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float ssqrt(float x) { return sqrtf(x); }
// The FP64 MUFU seeds flush subnormal inputs and results to zero (only .ftz
// variants exist), where the reference divides in IEEE: inputs whose
// reciprocal (or reciprocal root) would leave the normal range are scaled by a
// power of two first and the result scaled back (selects, no branch), so a
// subnormal pivot gives the finite IEEE quotient, not inf.
__device__ __forceinline__ double srcp(double x) {
  const double ax = fabs(x);
  const double s = ax < 0x1p-1000 ? 0x1p+64 : (ax > 0x1p+1000 ? 0x1p-64 : 1.0);
  const double xs = x * s;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(xs));
  double e = fma(-xs, r, 1.0);
  r = fma(r, e, r);
  e = fma(-xs, r, 1.0);
  return fma(r, e, r) * s;
}
__device__ __forceinline__ float srcp(float x) {
  float r;
  asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(x));  // no .ftz: subnormals kept
  return fmaf(r, fmaf(-x, r, 1.0f), r);
}
__device__ __forceinline__ double srsqrt(double x) {
  // x < 2^-1000: rsqrt(x 2^128) 2^64
  const bool tiny = x < 0x1p-1000;
  const double xs = tiny ? x * 0x1p+128 : x;
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(xs));
  const double h = 0.5 * xs;
  r = fma(r, fma(-h * r, r, 0.5), r);
  r = fma(r, fma(-h * r, r, 0.5), r);
  return tiny ? r * 0x1p+64 : r;
}
__device__ __forceinline__ float srsqrt(float x) {
  float r;
  asm("rsqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  const float h = 0.5f * x;
  return fmaf(r, fmaf(-h * r, r, 0.5f), r);
}
__device__ __forceinline__ double sfma(double a, double b, double c) {
  return fma(a, b, c);
}
__device__ __forceinline__ float sfma(float a, float b, float c) {
  return fmaf(a, b, c);
}

template <typename S, int R, int C>
__device__ __forceinline__ Mat<S, R, C> zeros() {
  Mat<S, R, C> m;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) m.a[i][j] = S(0);
  return m;
}
template <typename S, int N>
__device__ __forceinline__ Mat<S, N, N> eye() {
  Mat<S, N, N> m;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) m.a[i][j] = i == j ? S(1) : S(0);
  return m;
}

// ---- loads / stores (row-major, contiguous) ------------------------------
// Vectorised 16-byte accesses when the block is a multiple of 16 bytes; the
// host guarantees 16-byte alignment of every field base and step stride.
template <typename S, int R, int C>
__device__ __forceinline__ Mat<S, R, C> load(const S* __restrict__ p) {
  Mat<S, R, C> m;
  S* o = &m.a[0][0];
  constexpr int n = R * C;
  if constexpr ((n * sizeof(S)) % 16 == 0) {
    const float4* q = reinterpret_cast<const float4*>(p);
    constexpr int per = 16 / sizeof(S);
#pragma unroll
    for (int i = 0; i < n / per; ++i) {
      float4 v = __ldg(q + i);
      const S* vs = reinterpret_cast<const S*>(&v);
#pragma unroll
      for (int j = 0; j < per; ++j) o[i * per + j] = vs[j];
    }
  } else if constexpr ((n * sizeof(S)) % 8 == 0) {
    const float2* q = reinterpret_cast<const float2*>(p);
    constexpr int per = 8 / sizeof(S);
#pragma unroll
    for (int i = 0; i < n / per; ++i) {
      float2 v = __ldg(q + i);
      const S* vs = reinterpret_cast<const S*>(&v);
#pragma unroll
      for (int j = 0; j < per; ++j) o[i * per + j] = vs[j];
    }
  } else {
#pragma unroll
    for (int i = 0; i < n; ++i) o[i] = __ldg(p + i);
  }
  return m;
}
template <typename S, int R, int C>
__device__ __forceinline__ void store(S* __restrict__ p, const Mat<S, R, C>& m) {
  const S* o = &m.a[0][0];
  constexpr int n = R * C;
  if constexpr ((n * sizeof(S)) % 16 == 0) {
    float4* q = reinterpret_cast<float4*>(p);
    constexpr int per = 16 / sizeof(S);
#pragma unroll
    for (int i = 0; i < n / per; ++i) {
      float4 v;
      S* vs = reinterpret_cast<S*>(&v);
#pragma unroll
      for (int j = 0; j < per; ++j) vs[j] = o[i * per + j];
      __stcs(q + i, v);
    }
  } else if constexpr ((n * sizeof(S)) % 8 == 0) {
    float2* q = reinterpret_cast<float2*>(p);
    constexpr int per = 8 / sizeof(S);
#pragma unroll
    for (int i = 0; i < n / per; ++i) {
      float2 v;
      S* vs = reinterpret_cast<S*>(&v);
#pragma unroll
      for (int j = 0; j < per; ++j) vs[j] = o[i * per + j];
      __stcs(q + i, v);
    }
  } else {
#pragma unroll
    for (int i = 0; i < n; ++i) p[i] = o[i];
  }
}
// strided (SoA) access: element i of component c at p[c * stride]
template <typename S, int R, int C>
__device__ __forceinline__ Mat<S, R, C> load_soa(const S* p, size_t stride) {
  Mat<S, R, C> m;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) m.a[i][j] = p[(size_t)(i * C + j) * stride];
  return m;
}
template <typename S, int R, int C>
__device__ __forceinline__ void store_soa(S* p, size_t stride,
                                          const Mat<S, R, C>& m) {
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) p[(size_t)(i * C + j) * stride] = m.a[i][j];
}

// ---- products (mat.hpp:101-114 semantics, FMA accumulation) ---------------
template <typename S, int R, int K, int C>
__device__ __forceinline__ Mat<S, R, C> mul(const Mat<S, R, K>& x,
                                            const Mat<S, K, C>& y) {
  Mat<S, R, C> o;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      S acc = x.a[i][0] * y.a[0][j];
#pragma unroll
      for (int k = 1; k < K; ++k) acc = sfma(x.a[i][k], y.a[k][j], acc);
      o.a[i][j] = acc;
    }
  return o;
}
// x^T y
template <typename S, int K, int R, int C>
__device__ __forceinline__ Mat<S, R, C> mul_tn(const Mat<S, K, R>& x,
                                               const Mat<S, K, C>& y) {
  Mat<S, R, C> o;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      S acc = x.a[0][i] * y.a[0][j];
#pragma unroll
      for (int k = 1; k < K; ++k) acc = sfma(x.a[k][i], y.a[k][j], acc);
      o.a[i][j] = acc;
    }
  return o;
}
// symmetric result x y^T + z, upper triangle computed and mirrored (the
// mirror replaces the reference's mat_symmetrize, mat.hpp:124-136)
template <typename S, int N, int K>
__device__ __forceinline__ Mat<S, N, N> mul_nt_sym_add(const Mat<S, N, K>& x,
                                                       const Mat<S, N, K>& y,
                                                       const Mat<S, N, N>& z) {
  Mat<S, N, N> o;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i; j < N; ++j) {
      S acc = z.a[i][j];
#pragma unroll
      for (int k = 0; k < K; ++k) acc = sfma(x.a[i][k], y.a[j][k], acc);
      o.a[i][j] = acc;
      o.a[j][i] = acc;
    }
  return o;
}
// symmetric x^T y + z (upper triangle, mirrored)
template <typename S, int K, int N>
__device__ __forceinline__ Mat<S, N, N> mul_tn_sym_add(const Mat<S, K, N>& x,
                                                       const Mat<S, K, N>& y,
                                                       const Mat<S, N, N>& z) {
  Mat<S, N, N> o;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i; j < N; ++j) {
      S acc = z.a[i][j];
#pragma unroll
      for (int k = 0; k < K; ++k) acc = sfma(x.a[k][i], y.a[k][j], acc);
      o.a[i][j] = acc;
      o.a[j][i] = acc;
    }
  return o;
}
// x y + z
template <typename S, int R, int K, int C>
__device__ __forceinline__ Mat<S, R, C> mul_add(const Mat<S, R, K>& x,
                                                const Mat<S, K, C>& y,
                                                const Mat<S, R, C>& z) {
  Mat<S, R, C> o;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      S acc = z.a[i][j];
#pragma unroll
      for (int k = 0; k < K; ++k) acc = sfma(x.a[i][k], y.a[k][j], acc);
      o.a[i][j] = acc;
    }
  return o;
}
// z - x y
template <typename S, int R, int K, int C>
__device__ __forceinline__ Mat<S, R, C> sub_mul(const Mat<S, R, C>& z,
                                                const Mat<S, R, K>& x,
                                                const Mat<S, K, C>& y) {
  Mat<S, R, C> o;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      S acc = z.a[i][j];
#pragma unroll
      for (int k = 0; k < K; ++k) acc = sfma(-x.a[i][k], y.a[k][j], acc);
      o.a[i][j] = acc;
    }
  return o;
}
// z - x^T y
template <typename S, int K, int R, int C>
__device__ __forceinline__ Mat<S, R, C> sub_mul_tn(const Mat<S, R, C>& z,
                                                   const Mat<S, K, R>& x,
                                                   const Mat<S, K, C>& y) {
  Mat<S, R, C> o;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      S acc = z.a[i][j];
#pragma unroll
      for (int k = 0; k < K; ++k) acc = sfma(-x.a[k][i], y.a[k][j], acc);
      o.a[i][j] = acc;
    }
  return o;
}
// x^T y + z
template <typename S, int K, int R, int C>
__device__ __forceinline__ Mat<S, R, C> mul_tn_add(const Mat<S, K, R>& x,
                                                   const Mat<S, K, C>& y,
                                                   const Mat<S, R, C>& z) {
  Mat<S, R, C> o;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      S acc = z.a[i][j];
#pragma unroll
      for (int k = 0; k < K; ++k) acc = sfma(x.a[k][i], y.a[k][j], acc);
      o.a[i][j] = acc;
    }
  return o;
}
template <typename S, int R, int C>
__device__ __forceinline__ Mat<S, R, C> add(const Mat<S, R, C>& x,
                                            const Mat<S, R, C>& y) {
  Mat<S, R, C> o;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) o.a[i][j] = x.a[i][j] + y.a[i][j];
  return o;
}
template <typename S, int R, int C>
__device__ __forceinline__ Mat<S, R, C> sub(const Mat<S, R, C>& x,
                                            const Mat<S, R, C>& y) {
  Mat<S, R, C> o;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) o.a[i][j] = x.a[i][j] - y.a[i][j];
  return o;
}
template <typename S, int R, int C>
__device__ __forceinline__ Mat<S, C, R> trans(const Mat<S, R, C>& x) {
  Mat<S, C, R> o;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) o.a[j][i] = x.a[i][j];
  return o;
}
// (x + x^T)/2 (mat.hpp:124-136)
template <typename S, int N>
__device__ __forceinline__ void symmetrize(Mat<S, N, N>& x) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i + 1; j < N; ++j) {
      S m = (x.a[i][j] + x.a[j][i]) * S(0.5);
      x.a[i][j] = m;
      x.a[j][i] = m;
    }
}

// ---- Cholesky (mat.hpp:153-175) with reciprocal pivots --------------------
template <typename S, int N>
struct Chol {
  Mat<S, N, N> l;  // lower factor (strict upper unused)
  S inv[N];        // 1 / l(i,i)
};
template <typename S, int N>
__device__ __forceinline__ Chol<S, N> cholesky(const Mat<S, N, N>& a,
                                               unsigned& err) {
  Chol<S, N> c;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    S diag = a.a[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) diag = sfma(-c.l.a[j][k], c.l.a[j][k], diag);
    if (!(diag > S(0))) err |= kErrNotPD;
    const S il = srsqrt(diag);  // 1 / l(j,j)
    const S ljj = diag * il;
    c.l.a[j][j] = ljj;
    c.inv[j] = il;
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      S acc = a.a[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) acc = sfma(-c.l.a[i][k], c.l.a[j][k], acc);
      c.l.a[i][j] = acc * il;
    }
  }
  return c;
}
// X = A^{-1} B for A = L L^T (mat.hpp:244-269)
template <typename S, int N, int C>
__device__ __forceinline__ Mat<S, N, C> chol_solve(const Chol<S, N>& c,
                                                   const Mat<S, N, C>& b) {
  Mat<S, N, C> x;
#pragma unroll
  for (int col = 0; col < C; ++col) {
    S y[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      S acc = b.a[i][col];
#pragma unroll
      for (int k = 0; k < i; ++k) acc = sfma(-c.l.a[i][k], y[k], acc);
      y[i] = acc * c.inv[i];
    }
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
      S acc = y[i];
#pragma unroll
      for (int k = i + 1; k < N; ++k) acc = sfma(-c.l.a[k][i], y[k], acc);
      y[i] = acc * c.inv[i];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) x.a[i][col] = y[i];
  }
  return x;
}

// ---- LU with partial pivoting (mat.hpp:177-228) --------------------------
// Row swaps are applied with predicated moves; `piv[c]` is the row swapped
// into position c at step c (first maximum of |a(r,c)|, as the reference).
template <typename S, int N>
struct LU {
  Mat<S, N, N> a;  // unit-lower L below the diagonal, U on/above
  S inv[N];        // 1 / U(i,i)
  int piv[N];
};
template <typename S, int N>
__device__ __forceinline__ LU<S, N> lu_factor(const Mat<S, N, N>& m,
                                              unsigned& err) {
  LU<S, N> f;
  f.a = m;
#pragma unroll
  for (int c = 0; c < N; ++c) {
    S best = sabs(f.a.a[c][c]);
    int p = c;
#pragma unroll
    for (int r = c + 1; r < N; ++r) {
      S x = sabs(f.a.a[r][c]);
      bool gt = x > best;
      best = gt ? x : best;
      p = gt ? r : p;
    }
    f.piv[c] = p;
#pragma unroll
    for (int r = c + 1; r < N; ++r) {
      bool sw = (p == r);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        S t = f.a.a[c][j];
        S u = f.a.a[r][j];
        f.a.a[c][j] = sw ? u : t;
        f.a.a[r][j] = sw ? t : u;
      }
    }
    if (best == S(0)) err |= kErrSingular;
    S ip = srcp(f.a.a[c][c]);
    f.inv[c] = ip;
#pragma unroll
    for (int r = c + 1; r < N; ++r) {
      S fac = f.a.a[r][c] * ip;
      f.a.a[r][c] = fac;
#pragma unroll
      for (int j = c + 1; j < N; ++j)
        f.a.a[r][j] = sfma(-fac, f.a.a[c][j], f.a.a[r][j]);
    }
  }
  return f;
}
// X = M^{-1} B
template <typename S, int N, int C>
__device__ __forceinline__ Mat<S, N, C> lu_solve(const LU<S, N>& f,
                                                 const Mat<S, N, C>& b) {
  Mat<S, N, C> x;
#pragma unroll
  for (int col = 0; col < C; ++col) {
    S y[N];
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = b.a[i][col];
    // apply the row interchanges in factorisation order
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
      for (int r = c + 1; r < N; ++r) {
        bool sw = f.piv[c] == r;
        S t = y[c], u = y[r];
        y[c] = sw ? u : t;
        y[r] = sw ? t : u;
      }
#pragma unroll
    for (int i = 1; i < N; ++i)
#pragma unroll
      for (int k = 0; k < i; ++k) y[i] = sfma(-f.a.a[i][k], y[k], y[i]);
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
      S acc = y[i];
#pragma unroll
      for (int k = i + 1; k < N; ++k) acc = sfma(-f.a.a[i][k], y[k], acc);
      y[i] = acc * f.inv[i];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) x.a[i][col] = y[i];
  }
  return x;
}
// X = M^{-T} B  (M = P^T L U  =>  M^T = U^T L^T P)
template <typename S, int N, int C>
__device__ __forceinline__ Mat<S, N, C> lu_solve_t(const LU<S, N>& f,
                                                   const Mat<S, N, C>& b) {
  Mat<S, N, C> x;
#pragma unroll
  for (int col = 0; col < C; ++col) {
    S y[N];
    // U^T z = b (forward)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      S acc = b.a[i][col];
#pragma unroll
      for (int k = 0; k < i; ++k) acc = sfma(-f.a.a[k][i], y[k], acc);
      y[i] = acc * f.inv[i];
    }
    // L^T w = z (backward, unit diagonal)
#pragma unroll
    for (int i = N - 1; i >= 0; --i)
#pragma unroll
      for (int k = i + 1; k < N; ++k) y[i] = sfma(-f.a.a[k][i], y[k], y[i]);
    // x = P^T w : undo the interchanges in reverse order
#pragma unroll
    for (int c = N - 1; c >= 0; --c)
#pragma unroll
      for (int r = N - 1; r > c; --r) {
        bool sw = f.piv[c] == r;
        S t = y[c], u = y[r];
        y[c] = sw ? u : t;
        y[r] = sw ? t : u;
      }
#pragma unroll
    for (int i = 0; i < N; ++i) x.a[i][col] = y[i];
  }
  return x;
}

}  // namespace psk
