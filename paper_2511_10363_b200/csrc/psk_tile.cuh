// psk_tile.cuh -- register-tiled warp kernels for compile-time state and
// measurement dimensions up to the reference's kMaxDim = 16 (mat.hpp:19):
// BASELINE configs[4] (nx = 16, ny = 8) and the other (NX, NY) instantiated
// in psk_tile_impl.cuh.
//
// One warp per chunk, the formulation of psk_fast.cuh / psk_wide.cuh
// (chunked conditional-Kalman reduce, scan of chunk elements, finish that
// writes the per-step smoothing elements, smoother finish).  What changes
// against the runtime-dimension wide path is how a warp does a small matrix
// product: every product is a compile-time (M x N x K) warp GEMM in which
// lane l owns a TM x TN tile of the output in REGISTERS (8-16 independent FMA
// chains), operands stream from shared memory as 16-byte vector loads laid
// out so that lanes sharing a row (column) of the tile read the same address
// (shared-memory broadcast), and the result is written back once.  Matrices
// are stored row-major or column-major, whichever makes the next product's
// operand a contiguous vector; rows are padded to LD = N + 2 scalars so the
// transposed reads of output stores stay (nearly) conflict-free.  Solves are
// Gauss-Jordan eliminations with one column per lane in registers and the
// pivot column broadcast through shared memory (SPD blocks: no pivoting, a
// non-positive pivot raises kErrNotPD as the reference's Cholesky does,
// mat.hpp:165).  Everything is fully unrolled: no runtime index arithmetic,
// no divisions, no spills.
//
// Symmetric results (C, J, P, PP, S, L) are stored from the upper triangle
// of the product and mirrored (put_sym), so every symmetric matrix stays
// exactly symmetric like the reference's (mat_symmetrize, mat.hpp:126-136).
#pragma once
#include <cuda_runtime.h>

#include "psk_common.cuh"
#include "psk_mat.cuh"

namespace psk {
namespace tile {

// Lanes per chunk: a HALF warp works on one chunk, so every warp carries two
// chunks and a 16 x 16 product gives each lane a 4 x 4 tile (0.5 operand
// loads per FMA instead of 0.75 for 2 x 4 tiles on a full warp -- the kernels
// are bound by shared-memory -> register bandwidth).
constexpr int kGW = 16;
// lane within the chunk's group, the group's mask, group-wide sync
__device__ __forceinline__ int lane() { return threadIdx.x & (kGW - 1); }
__device__ __forceinline__ unsigned gmask() {
  return kGW == 32 ? 0xffffffffu : (((1u << kGW) - 1u) << (threadIdx.x & 31 & ~(kGW - 1)));
}
__device__ __forceinline__ void gsync() { __syncwarp(gmask()); }

template <typename S>
constexpr int vec16() {
  return 16 / (int)sizeof(S);
}
// round n scalars up to whole 16-byte units
template <typename S>
constexpr int up16(int n) {
  return (n + vec16<S>() - 1) / vec16<S>() * vec16<S>();
}

// v[i] = p[i * ST], i < n: 16-byte vector loads when contiguous
template <int n, int ST, typename S>
__device__ __forceinline__ void ld(S (&v)[n], const S* p) {
  if constexpr (ST == 1 && (n * (int)sizeof(S)) % 16 == 0) {
#pragma unroll
    for (int i = 0; i < n * (int)sizeof(S) / 16; ++i) {
      const float4 q = *reinterpret_cast<const float4*>(p + i * vec16<S>());
      const S* qs = reinterpret_cast<const S*>(&q);
#pragma unroll
      for (int j = 0; j < vec16<S>(); ++j) v[i * vec16<S>() + j] = qs[j];
    }
  } else if constexpr (ST == 1 && n * (int)sizeof(S) == 8) {
    const float2 q = *reinterpret_cast<const float2*>(p);
    const S* qs = reinterpret_cast<const S*>(&q);
#pragma unroll
    for (int j = 0; j < n; ++j) v[j] = qs[j];
  } else {
#pragma unroll
    for (int i = 0; i < n; ++i) v[i] = p[i * ST];
  }
}
template <int n, int ST, typename S>
__device__ __forceinline__ void st(S* p, const S (&v)[n]) {
  if constexpr (ST == 1 && (n * (int)sizeof(S)) % 16 == 0) {
#pragma unroll
    for (int i = 0; i < n * (int)sizeof(S) / 16; ++i) {
      float4 q;
      S* qs = reinterpret_cast<S*>(&q);
#pragma unroll
      for (int j = 0; j < vec16<S>(); ++j) qs[j] = v[i * vec16<S>() + j];
      *reinterpret_cast<float4*>(p + i * vec16<S>()) = q;
    }
  } else if constexpr (ST == 1 && n * (int)sizeof(S) == 8) {
    float2 q;
    S* qs = reinterpret_cast<S*>(&q);
#pragma unroll
    for (int j = 0; j < n; ++j) qs[j] = v[j];
    *reinterpret_cast<float2*>(p) = q;
  } else {
#pragma unroll
    for (int i = 0; i < n; ++i) p[i * ST] = v[i];
  }
}

// Output tiling of an M x N result over the chunk's lane group: lane -> tile
// (tr, tc) of TM x TN; lanes >= TR * TC hold no tile.
template <int M, int N, int TM, int TN>
struct Tiling {
  static constexpr int TR = M / TM, TC = N / TN, tiles = TR * TC;
  static_assert(M % TM == 0 && N % TN == 0 && tiles <= kGW, "tiling");
  __device__ __forceinline__ static bool active() { return tiles == kGW || lane() < tiles; }
  __device__ __forceinline__ static int r0() { return (lane() / TC) * TM; }
  __device__ __forceinline__ static int c0() { return (lane() % TC) * TN; }
};

// acc(i, j) += sum_k L(r0 + i, k) R(k, c0 + j), L(r, k) at lp[r LR + k LK],
// R(k, c) at rp[k RK + c RC]; lp / rp already offset to (r0, 0) / (0, c0).
// (NEG: acc -= ...)
template <int K, int TM, int TN, int LR, int LK, int RK, int RC, bool NEG = false, typename S>
__device__ __forceinline__ void mma(S (&acc)[TM][TN], const S* lp, const S* rp) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    S a[TM], b[TN];
    ld<TM, LR>(a, lp + k * LK);
    ld<TN, RC>(b, rp + k * RK);
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = sfma(NEG ? -a[i] : a[i], b[j], acc[i][j]);
  }
}
template <int TM, int TN, typename S>
__device__ __forceinline__ void zero(S (&acc)[TM][TN]) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = S(0);
}
// acc(i, j) = Z(r0 + i, c0 + j) (Z(r, c) at z[r ZR + c ZC])
template <int TM, int TN, int ZR, int ZC, typename S>
__device__ __forceinline__ void init(S (&acc)[TM][TN], const S* z) {
  if constexpr (ZC == 1) {
#pragma unroll
    for (int i = 0; i < TM; ++i) ld<TN, 1>(acc[i], z + i * ZR);
  } else {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = z[i * ZR + j * ZC];
  }
}
// O(r0 + i, c0 + j) = acc(i, j), O(r, c) at o[r OR + c OC]
template <int TM, int TN, int OR, int OC, typename S>
__device__ __forceinline__ void put(S* o, const S (&acc)[TM][TN]) {
  if constexpr (OC == 1) {
#pragma unroll
    for (int i = 0; i < TM; ++i) st<TN, 1>(o + i * OR, acc[i]);
  } else if constexpr (OR == 1) {
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      S col[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i) col[i] = acc[i][j];
      st<TM, 1>(o + j * OC, col);
    }
  } else {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) o[i * OR + j * OC] = acc[i][j];
  }
}
// Symmetric result: the upper-triangle entries of the tile (c >= r) are
// stored at (r, c) and mirrored to (c, r); lower entries are dropped (their
// mirror images come from the lanes owning the upper ones).  Exactly
// symmetric like the reference's symmetrised products (mat.hpp:126-136) --
// the unsymmetrised recursion loses definiteness over long chunks.
template <int TM, int TN, int OR, typename S>
__device__ __forceinline__ void put_sym(S* o, const S (&acc)[TM][TN], int r0, int c0) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int r = r0 + i, c = c0 + j;
      if (c >= r) {
        o[r * OR + c] = acc[i][j];
        o[c * OR + r] = acc[i][j];
      }
    }
}
template <int TM, int TN, typename S>
__device__ __forceinline__ void neg(S (&acc)[TM][TN]) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = -acc[i][j];
}

// Gauss-Jordan elimination without pivoting on the R x W block X (row stride
// LDX): [A | B] -> [I | A^-1 B] for A symmetric positive definite.  Lane l
// of the group holds columns l, l + kGW, ... in registers; the pivot column is published by
// its owner lane through pv (2 R scalars, double-buffered) and read back by
// every lane as broadcast vector loads.
template <int R, int W, int LDX, typename S>
__device__ __forceinline__ void gj_spd(S* X, S* pv, unsigned& err) {
  constexpr int NC = (W + kGW - 1) / kGW;
  static_assert(R <= kGW, "pivot column owner");
  const int ln = lane();
  S x[NC][R];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int col = ln + kGW * c;
#pragma unroll
    for (int i = 0; i < R; ++i) x[c][i] = col < W ? X[i * LDX + col] : S(0);
  }
#pragma unroll
  for (int p = 0; p < R; ++p) {
    S* buf = pv + (p & 1) * R;
    if (ln == p) st<R, 1>(buf, x[0]);
    gsync();
    S col[R];
    ld<R, 1>(col, buf);
    const S d = col[p];
    if (!(d > S(0))) err |= kErrNotPD;
    const S ip = srcp(d);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const S rp = x[c][p] * ip;
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (i != p) x[c][i] = sfma(-col[i], rp, x[c][i]);
      x[c][p] = rp;
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int col = ln + kGW * c;
    if (col < W) {
#pragma unroll
      for (int i = 0; i < R; ++i) X[i * LDX + col] = x[c][i];
    }
  }
  gsync();
}

// Gauss-Jordan elimination WITH partial pivoting (the reference's pivoted LU,
// mat.hpp:180-205: first maximum |a(r, p)| over r >= p) on the R x W block
// X: [A | B] -> [I | A^-1 B] for a general nonsingular A (a zero pivot
// raises kErrSingular).  Same layout as gj_spd; the pivot row is found by the
// owner of column p and broadcast to the group with a shuffle, and every lane
// swaps rows p and pr of its columns in registers (predicated, static
// indices).
template <int R, int W, int LDX, typename S>
__device__ __forceinline__ void gj_piv(S* X, S* pv, unsigned& err) {
  constexpr int NC = (W + kGW - 1) / kGW;
  static_assert(R <= kGW, "pivot column owner");
  const int ln = lane();
  const int base = threadIdx.x & 31 & ~(kGW - 1);
  S x[NC][R];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int col = ln + kGW * c;
#pragma unroll
    for (int i = 0; i < R; ++i) x[c][i] = col < W ? X[i * LDX + col] : S(0);
  }
#pragma unroll
  for (int p = 0; p < R; ++p) {
    S best = S(-1);
    int pr = p;
#pragma unroll
    for (int i = p; i < R; ++i)
      if (sabs(x[0][i]) > best) {
        best = sabs(x[0][i]);
        pr = i;
      }
    pr = __shfl_sync(gmask(), pr, base + p);
    if (pr != p) {  // group-uniform: swap rows p and pr in every column
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const S a = x[c][p];
#pragma unroll
        for (int i = p + 1; i < R; ++i)
          if (i == pr) {
            x[c][p] = x[c][i];
            x[c][i] = a;
          }
      }
    }
    S* buf = pv + (p & 1) * R;
    if (ln == p) st<R, 1>(buf, x[0]);
    gsync();
    S col[R];
    ld<R, 1>(col, buf);
    const S d = col[p];
    if (d == S(0)) err |= kErrSingular;
    const S ip = srcp(d);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const S rp = x[c][p] * ip;
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (i != p) x[c][i] = sfma(-col[i], rp, x[c][i]);
      x[c][p] = rp;
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int col = ln + kGW * c;
    if (col < W) {
#pragma unroll
      for (int i = 0; i < R; ++i) X[i * LDX + col] = x[c][i];
    }
  }
  gsync();
}

// y(r) = sum_k A(r, k) x(k) (+ z(r)), A(r, k) at a[r AR + k AK]; lanes r < n
template <int n, int K, int AR, int AK, typename S>
__device__ __forceinline__ S matvec_row(const S* a, const S* x, int r) {
  S acc0 = S(0), acc1 = S(0);
#pragma unroll
  for (int k = 0; k < K; k += 2) {
    acc0 = sfma(a[r * AR + k * AK], x[k], acc0);
    if (k + 1 < K) acc1 = sfma(a[r * AR + (k + 1) * AK], x[k + 1], acc1);
  }
  return acc0 + acc1;
}

// ---- frames -------------------------------------------------------------------
// Model blocks of one step in shared memory, laid out for the products:
// F column-major (F(r, c) at Fc[c LD + r]), Q row-major, H transposed
// (H(r, c) at Ht[c LDM + r]), R row-major, vectors u, d, y.
// row stride of an N-column matrix: 16-byte rows, padded by at least one
// scalar so that column walks do not all hit one bank
template <typename S>
constexpr int ldpad(int n) {
  return up16<S>(n + 1);
}
template <typename S, int N, int M>
struct ModelFrame {
  static constexpr int LD = ldpad<S>(N), LDM = ldpad<S>(M), LDR = ldpad<S>(M);
  static constexpr int Fc = 0, Q = up16<S>(N * LD), Ht = Q + up16<S>(N * LD),
                       R = Ht + up16<S>(N * LDM), u = R + up16<S>(M * LDR), d = u + up16<S>(N),
                       y = d + up16<S>(M), size = y + up16<S>(M);
};

// load step k's blocks (all of them, or only F, Q, u) from global memory
template <typename S, int N, int M>
__device__ __forceinline__ void load_model(S* mf, const ModelView<S>& m, long long k,
                                           bool fqu_only = false) {
  using MF = ModelFrame<S, N, M>;
  const int ln = lane();
  const S* F = m.F(k);
  const S* Q = m.Q(k);
#pragma unroll
  for (int i = ln; i < N * N; i += kGW) {
    const int r = i / N, c = i % N;
    mf[MF::Fc + c * MF::LD + r] = F[i];
    mf[MF::Q + r * MF::LD + c] = Q[i];
  }
  if (ln < N) mf[MF::u + ln] = m.U(k)[ln];
  if (fqu_only) return;
  const S* H = m.H(k);
#pragma unroll
  for (int i = ln; i < M * N; i += kGW) {
    const int r = i / N, c = i % N;
    mf[MF::Ht + c * MF::LDM + r] = H[i];
  }
  const S* Rg = m.R(k);
#pragma unroll
  for (int i = ln; i < M * M; i += kGW) mf[MF::R + (i / M) * MF::LDR + (i % M)] = Rg[i];
  if (ln < M) {
    mf[MF::d + ln] = m.D(k)[ln];
    mf[MF::y + ln] = m.Y(k)[ln];
  }
}

// The model frame of a warp: one CTA-wide copy when F, Q, H, R, u, d are all
// time-invariant (stride 0: loaded once, y read per step), else one per warp
// refilled every step.
template <typename S>
__host__ __device__ __forceinline__ bool time_invariant(const ModelView<S>& m) {
  return m.sf == 0 && m.sq == 0 && m.sh == 0 && m.sr == 0 && m.su == 0 && m.sd == 0;
}

// Store the N x N matrix at a (row stride LDa, column-major if COLM) to global
// g[r N + c] (coalesced); SYM: take the upper triangle for both halves.
template <int N, int LDa, bool COLM, bool SYM, typename S>
__device__ __forceinline__ void gstore_mat(S* g, const S* a) {
#pragma unroll
  for (int i = lane(); i < N * N; i += kGW) {
    int r = i / N, c = i % N;
    if (SYM && r > c) {
      const int t = r;
      r = c;
      c = t;
    }
    g[i] = COLM ? a[c * LDa + r] : a[r * LDa + c];
  }
}
template <int N, int LDa, bool COLM, typename S>
__device__ __forceinline__ void sload_mat(S* a, const S* g) {
#pragma unroll
  for (int i = lane(); i < N * N; i += kGW) {
    const int r = i / N, c = i % N;
    if (COLM)
      a[c * LDa + r] = g[i];
    else
      a[r * LDa + c] = g[i];
  }
}

}  // namespace tile
}  // namespace psk
