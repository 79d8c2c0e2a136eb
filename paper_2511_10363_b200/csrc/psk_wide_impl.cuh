// psk_wide_impl.cuh -- warp-per-chunk kernels, scan operators and host
// dispatch of the wide fast path (psk_wide.cuh): runtime nx, ny <= 16.
//
// Same formulation and launch sequence as the register-resident path
// (psk_fast.cuh / psk_fast_impl.cuh), one warp in place of one thread:
//   reduce (conditional Kalman)  ->  chunk scan  ->  finish (filtered stats,
//   or per-step smoothing elements + smoother chunk fold)  ->  reverse chunk
//   scan  ->  smoother finish.
// Chunk elements are stored AoS (element i at p + i * ES: a warp reads an
// element with one coalesced sweep).  The chunk scans run the reference's
// level-by-level index maps with one warp per combine (k_level<Ops, 32>);
// the decoupled look-back request maps to the Ladner-Fischer plan here.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>

#include "psk_exact.h"
#include "psk_levels.cuh"
#include "psk_plan.hpp"
#include "psk_wide.cuh"

namespace psk {
namespace wide {

// ---- per-warp shared-memory slots ---------------------------------------
template <typename S>
struct Slots {
  S* base;
  int nm;  // matrix slots before the vectors
  __device__ __forceinline__ S* m(int i) const { return base + i * kMat; }
  __device__ __forceinline__ S* v(int i) const { return base + nm * kMat + i * kVec; }
  __device__ __forceinline__ int* piv() const {
    return reinterpret_cast<int*>(base + nm * kMat + 14 * kVec);
  }
};
// every kernel / operator below uses at most this many slots per warp
constexpr int kMatSlots = 14;
constexpr int kVecSlots = 16;  // the last two hold pivots
template <typename S>
constexpr int warp_bytes() {
  return (kMatSlots * kMat + kVecSlots * kVec) * (int)sizeof(S);
}
template <typename S>
__device__ __forceinline__ Slots<S> warp_slots(int nm = kMatSlots) {
  extern __shared__ __align__(16) unsigned char wsm[];
  S* base = reinterpret_cast<S*>(wsm) + (threadIdx.x >> 5) * (nm * kMat + kVecSlots * kVec);
  return Slots<S>{base, nm};
}
// Matrix slots of the per-step kernels: A, C, J, 7 scratch, plus one per
// model matrix (F, Q, H, R) that varies with the step -- a time-invariant
// (stride-0) matrix is read in place from global memory (L1-resident), which
// frees its slot: BASELINE configs[4]'s broadcast models run 10 slots/warp.
// (FP64 only: FP32 slots are half the size and occupancy is set by
// registers, so FP32 keeps every matrix in shared memory.)
template <typename S>
__host__ __device__ __forceinline__ bool staged_input(long long stride) {
  return stride != 0 || sizeof(S) == 4;
}
template <typename S>
__host__ __device__ __forceinline__ int step_slots(const ModelView<S>& m) {
  return 10 + staged_input<S>(m.sf) + staged_input<S>(m.sq) + staged_input<S>(m.sh) +
         staged_input<S>(m.sr);
}
template <typename S>
__host__ __device__ __forceinline__ int step_smem(int nm) {
  return kWarps * (nm * kMat + kVecSlots * kVec) * (int)sizeof(S);
}

template <typename S>
__device__ __forceinline__ void vadd(WM<S> o, WM<S> a, WM<S> b, int n, S sb) {
  for (int i = lane_id(); i < n; i += 32) o(i, 0) = sfma(sb, b(i, 0), a(i, 0));
  __syncwarp();
}
template <typename S>
__device__ __forceinline__ void add_eye(WM<S> a, int n) {
  for (int i = lane_id(); i < n; i += 32) a(i, i) += S(1);
  __syncwarp();
}

// ---- element layout (AoS, FLayout / SLayout order, runtime n) ------------
struct FOffs {
  int A, b, C, eta, J, size;
  __host__ __device__ explicit FOffs(int n)
      : A(0), b(n * n), C(n * n + n), eta(2 * n * n + n), J(2 * n * n + 2 * n),
        size(3 * n * n + 2 * n) {}
};
struct SOffs {
  int E, g, L, size;
  __host__ __device__ explicit SOffs(int n)
      : E(0), g(n * n), L(n * n + n), size(2 * n * n + n) {}
};

// ---- Lemma 1 (kalman_elems.hpp:267-336) on shared-memory operands --------
// l = (A,b,C,eta,J) earlier, r = later, o = result (o may not alias l, r);
// scratch: 4 matrix slots + 3 vector slots + pivots from `sc`.
template <typename S>
__device__ void filter_combine(S* o, const S* l, const S* r, int n, Slots<S> sc, int m0,
                               int v0, unsigned& err) {
  const FOffs F(n);
  auto M = [&](const S* p, int off) { return WM<S>{const_cast<S*>(p) + off, n}; };
  auto V = [&](const S* p, int off) { return WM<S>{const_cast<S*>(p) + off, 1}; };
  // [M | I] with M = I + C_l J_r (2 slots) -> [I | M^-1] by Gauss-Jordan with
  // partial pivoting; N = I + J_r C_l = M^T (C, J symmetric), so
  // N^-1 = (M^-1)^T and every solve of Lemma 1 becomes a product
  WM<S> aug{sc.m(m0), 2 * n};
  WM<S> t1 = mat(sc.m(m0 + 2)), t2 = mat(sc.m(m0 + 3));
  WM<S> u1 = vec(sc.v(v0 + 1)), u2 = vec(sc.v(v0 + 2));
  gemm<false, false>(aug, M(l, F.C), M(r, F.J), n, n, n);
  for_each(n, n, [&](int i, int j) {
    aug(i, n + j) = i == j ? S(1) : S(0);
    if (i == j) aug(i, i) += S(1);
  });
  __syncwarp();
  gauss_jordan(aug, n, 2 * n, true, err);
  const WM<S> Mi{aug.p + n, 2 * n};
  // A' = A_r M^-1 A_l
  gemm<false, false>(t1, Mi, M(l, F.A), n, n, n);
  gemm<false, false>(M(o, F.A), M(r, F.A), t1, n, n, n);
  // b' = A_r M^-1 (C_l eta_r + b_l) + b_r
  gemm<false, false>(u1, M(l, F.C), V(r, F.eta), n, n, 1, l + F.b, 1);
  gemm<false, false>(u2, Mi, u1, n, n, 1);
  gemm<false, false>(V(o, F.b), M(r, F.A), u2, n, n, 1, r + F.b, 1);
  // C' = A_r M^-1 C_l A_r^T + C_r (symmetric)
  gemm<false, false>(t1, Mi, M(l, F.C), n, n, n);
  gemm<false, false>(t2, M(r, F.A), t1, n, n, n);
  gemm<false, true>(M(o, F.C), t2, M(r, F.A), n, n, n, r + F.C, n, S(1), true);
  // eta' = A_l^T M^-T (eta_r - J_r b_l) + eta_l
  gemm<false, false>(u1, M(r, F.J), V(l, F.b), n, n, 1, r + F.eta, 1, S(-1));
  gemm<true, false>(u2, Mi, u1, n, n, 1);
  gemm<true, false>(V(o, F.eta), M(l, F.A), u2, n, n, 1, l + F.eta, 1);
  // J' = A_l^T M^-T J_r A_l + J_l (symmetric)
  gemm<true, false>(t1, Mi, M(r, F.J), n, n, n);
  gemm<false, false>(t2, t1, M(l, F.A), n, n, n);
  gemm<true, false>(M(o, F.J), M(l, F.A), t2, n, n, n, l + F.J, n, S(1), true);
}
// Lemma 2 (kalman_elems.hpp:396-418): E' = E_l E_r, g' = E_l g_r + g_l,
// L' = E_l L_r E_l^T + L_l; scratch: 1 matrix slot
template <typename S>
__device__ void smoother_combine(S* o, const S* l, const S* r, int n, Slots<S> sc, int m0) {
  const SOffs F(n);
  auto M = [&](const S* p, int off) { return WM<S>{const_cast<S*>(p) + off, n}; };
  auto V = [&](const S* p, int off) { return WM<S>{const_cast<S*>(p) + off, 1}; };
  WM<S> t = mat(sc.m(m0));
  gemm<false, false>(M(o, F.E), M(l, F.E), M(r, F.E), n, n, n);
  gemm<false, false>(V(o, F.g), M(l, F.E), V(r, F.g), n, n, 1, l + F.g, 1);
  gemm<false, false>(t, M(l, F.E), M(r, F.L), n, n, n);
  gemm<false, true>(M(o, F.L), t, M(l, F.E), n, n, n, l + F.L, n, S(1), true);
}

// ---- scan operator policies (warp-cooperative, AoS global buffers) --------
// Operands are staged into the warp's slots (an element fits in 4 slots),
// combined, and the result written back: dst may alias an operand.
template <typename S_>
struct WideFilterOps {
  using S = S_;
  static constexpr int kSize = 0;  // runtime element size (AoS): unused by the level kernel
  unsigned* err;
  int n;
  __device__ void combine(const ElemBuf<S>& d, long long di, const ElemBuf<S>& l, long long li,
                          const ElemBuf<S>& r, long long ri) const {
    const Slots<S> sc = warp_slots<S>();
    const int es = FOffs(n).size;  // <= 800 = 2.94 slots
    S* sl = sc.m(0);
    S* sr = sc.m(3);
    S* so = sc.m(6);
    for (int i = lane_id(); i < es; i += 32) {
      sl[i] = l.p[li * es + i];
      sr[i] = r.p[ri * es + i];
    }
    __syncwarp();
    unsigned e = 0;
    filter_combine(so, sl, sr, n, sc, 9, 0, e);
    for (int i = lane_id(); i < es; i += 32) d.p[di * es + i] = so[i];
    __syncwarp();
    if (e && lane_id() == 0) atomicOr(err, e);
  }
  __device__ void assign(const ElemBuf<S>& d, long long di, const ElemBuf<S>& s,
                         long long si) const {
    const int es = FOffs(n).size;
    for (int i = lane_id(); i < es; i += 32) d.p[di * es + i] = s.p[si * es + i];
    __syncwarp();
  }
  __device__ void identity(const ElemBuf<S>& d, long long di) const {
    const FOffs F(n);
    for (int i = lane_id(); i < F.size; i += 32) {
      S v = S(0);
      if (i < F.b) v = (i / n == i % n) ? S(1) : S(0);
      d.p[di * F.size + i] = v;
    }
    __syncwarp();
  }
};
template <typename S_>
struct WideSmootherOps {
  using S = S_;
  static constexpr int kSize = 0;
  int n;
  __device__ void combine(const ElemBuf<S>& d, long long di, const ElemBuf<S>& l, long long li,
                          const ElemBuf<S>& r, long long ri) const {
    const Slots<S> sc = warp_slots<S>();
    const int es = SOffs(n).size;  // <= 528 = 1.94 slots
    S* sl = sc.m(0);
    S* sr = sc.m(2);
    S* so = sc.m(4);
    for (int i = lane_id(); i < es; i += 32) {
      sl[i] = l.p[li * es + i];
      sr[i] = r.p[ri * es + i];
    }
    __syncwarp();
    smoother_combine(so, sl, sr, n, sc, 6);
    for (int i = lane_id(); i < es; i += 32) d.p[di * es + i] = so[i];
    __syncwarp();
  }
  __device__ void assign(const ElemBuf<S>& d, long long di, const ElemBuf<S>& s,
                         long long si) const {
    const int es = SOffs(n).size;
    for (int i = lane_id(); i < es; i += 32) d.p[di * es + i] = s.p[si * es + i];
    __syncwarp();
  }
  __device__ void identity(const ElemBuf<S>& d, long long di) const {
    const SOffs F(n);
    for (int i = lane_id(); i < F.size; i += 32) {
      S v = S(0);
      if (i < F.g) v = (i / n == i % n) ? S(1) : S(0);
      d.p[di * F.size + i] = v;
    }
    __syncwarp();
  }
};

// ---- per-step building blocks ---------------------------------------------
// Shared-memory slots of the per-step kernels:
//   matrices 0 A | 1 C | 2 J | 3 F | 4 Q | 5 H | 6 R | 7..13 scratch
//   vectors  0 b | 1 eta | 2 u | 3 d | 4 y | 5..13 scratch, 14-15 pivots
template <typename S>
struct Step {
  Slots<S> sc;
  int nx, ny;
  const S *fg, *qg, *hg, *rg;  // broadcast model matrices in global memory
  int fs, qs, hs, rs;          // their slots when staged per step (-1: global)
  __device__ Step(const ModelView<S>& m, int nx_, int ny_)
      : sc(warp_slots<S>(step_slots(m))), nx(nx_), ny(ny_), fg(m.f), qg(m.q), hg(m.h),
        rg(m.r) {
    int k = 10;
    fs = staged_input<S>(m.sf) ? k++ : -1;
    qs = staged_input<S>(m.sq) ? k++ : -1;
    hs = staged_input<S>(m.sh) ? k++ : -1;
    rs = staged_input<S>(m.sr) ? k++ : -1;
  }
  __device__ WM<S> A() const { return mat(sc.m(0)); }
  __device__ WM<S> C() const { return mat(sc.m(1)); }
  __device__ WM<S> J() const { return mat(sc.m(2)); }
  __device__ WM<S> F() const { return fs >= 0 ? mat(sc.m(fs)) : WM<S>{const_cast<S*>(fg), nx}; }
  __device__ WM<S> Q() const { return qs >= 0 ? mat(sc.m(qs)) : WM<S>{const_cast<S*>(qg), nx}; }
  __device__ WM<S> H() const { return hs >= 0 ? mat(sc.m(hs)) : WM<S>{const_cast<S*>(hg), nx}; }
  __device__ WM<S> R() const { return rs >= 0 ? mat(sc.m(rs)) : WM<S>{const_cast<S*>(rg), ny}; }
  __device__ WM<S> T(int i) const { return mat(sc.m(3 + i)); }  // i < 7
  __device__ WM<S> b() const { return vec(sc.v(0)); }
  __device__ WM<S> eta() const { return vec(sc.v(1)); }
  __device__ WM<S> u() const { return vec(sc.v(2)); }
  __device__ WM<S> d() const { return vec(sc.v(3)); }
  __device__ WM<S> y() const { return vec(sc.v(4)); }
  __device__ WM<S> t(int i) const { return vec(sc.v(5 + i)); }  // i < 9
  // model blocks of step k (coalesced); broadcast matrices stay in place
  __device__ void load(const ModelView<S>& m, long long k) const {
    if (fs >= 0) gload(F(), m.F(k), nx, nx);
    if (qs >= 0) gload(Q(), m.Q(k), nx, nx);
    if (hs >= 0) gload(H(), m.H(k), ny, nx);
    if (rs >= 0) gload(R(), m.R(k), ny, ny);
    gload(u(), m.U(k), nx, 1);
    gload(d(), m.D(k), ny, 1);
    gload(y(), m.Y(k), ny, 1);
    __syncwarp();
  }
  // the transition of step k into the F / Q / u slots (chunk-end element)
  __device__ void load_fqu(const ModelView<S>& m, long long k) const {
    if (fs >= 0) gload(F(), m.F(k), nx, nx);
    if (qs >= 0) gload(Q(), m.Q(k), nx, nx);
    gload(u(), m.U(k), nx, 1);
    __syncwarp();
  }
};

// Conditional update of the running element (A, b, C, eta, J) with the
// measurement in `st` (the wide twin of psk_fast.cuh cond_update).
template <typename S>
__device__ void cond_update(const Step<S>& st, unsigned& err) {
  const int nx = st.nx, ny = st.ny;
  WM<S> hc = st.T(0), ha = st.T(4);
  WM<S> v = st.t(0);
  // [S | H C | H A | v] (<= 16 x 49, slots T1..T3) -> S^-1 [H C | H A | v]
  const int w = ny + 2 * nx + 1;
  WM<S> aug{st.T(1).p, w};
  WM<S> kt{aug.p + ny, w}, wm{aug.p + ny + nx, w}, sv{aug.p + ny + 2 * nx, w};
  gemm<false, false>(hc, st.H(), st.C(), ny, nx, nx);
  gemm<false, false>(ha, st.H(), st.A(), ny, nx, nx);
  gemm<false, false>(v, st.H(), st.b(), ny, nx, 1, st.y().p, 1, S(-1));
  vadd(v, v, st.d(), ny, S(-1));
  gemm<false, true>(aug, hc, st.H(), ny, nx, ny, st.R().p, st.R().ld, S(1), true);
  copy(kt, hc, ny, nx);
  copy(wm, ha, ny, nx);
  copy(sv, v, ny, 1);
  gauss_jordan(aug, ny, w, false, err);  // kt = K^T, wm = S^-1 H A, sv = S^-1 v
  gemm<true, false>(st.eta(), ha, sv, nx, ny, 1, st.eta().p, 1);
  gemm<true, false>(st.J(), ha, wm, nx, ny, nx, st.J().p, kLd, S(1), true);
  gemm<true, false>(st.A(), kt, ha, nx, ny, nx, st.A().p, kLd, S(-1));
  gemm<true, false>(st.b(), kt, v, nx, ny, 1, st.b().p, 1);
  gemm<true, false>(st.C(), kt, hc, nx, ny, nx, st.C().p, kLd, S(-1), true);
}

// ---- kernels ----------------------------------------------------------------
// reduce: chunk c -> one filtering element (AoS at agg + c * ES)
template <typename S>
__global__ void __launch_bounds__(32 * kWarps)
    k_wide_reduce(ModelView<S> m, long long L, long long nchunks, S* agg, unsigned* err) {
  const long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= nchunks) return;  // warp-uniform
  const int nx = m.nx, ny = m.ny;
  const Step<S> st(m, nx, ny);
  unsigned e = 0;
  const long long k0 = c * L, k1 = min(k0 + L, m.t);
  // identity, or the prior in state form for the chunk holding step 1
  // (kalman_elems.hpp:68-96; see k_filter_reduce)
  const bool prior = k0 == 0 && m.prior_first;
  fill(st.A(), nx, nx, prior ? S(0) : S(1), S(0));
  fill(st.J(), nx, nx, S(0), S(0));
  fill(st.eta(), nx, 1, S(0), S(0));
  if (prior) {
    gload(st.b(), m.m0, nx, 1);
    gload(st.C(), m.p0, nx, nx);
  } else {
    fill(st.b(), nx, 1, S(0), S(0));
    fill(st.C(), nx, nx, S(0), S(0));
  }
  __syncwarp();
  for (long long k = k0; k < k1; ++k) {
    st.load(m, k);
    // predict the conditional: (F A, F b + u, F C F^T + Q)
    gemm<false, false>(st.T(6), st.F(), st.A(), nx, nx, nx);
    copy(st.A(), st.T(6), nx, nx);
    gemm<false, false>(st.t(2), st.F(), st.b(), nx, nx, 1, st.u().p, 1);
    copy(st.b(), st.t(2), nx, 1);
    gemm<false, false>(st.T(6), st.F(), st.C(), nx, nx, nx);
    gemm<false, true>(st.C(), st.T(6), st.F(), nx, nx, nx, st.Q().p, st.Q().ld, S(1), true);
    cond_update(st, e);
  }
  const FOffs F(nx);
  S* o = agg + c * F.size;
  gstore(o + F.A, st.A(), nx, nx);
  gstore(o + F.b, st.b(), nx, 1);
  gstore(o + F.C, st.C(), nx, nx);
  gstore(o + F.eta, st.eta(), nx, 1);
  gstore(o + F.J, st.J(), nx, nx);
  if (e && lane_id() == 0) atomicOr(err, e);
}

// Smoothing element of step k-1 from its filtered (x, P) (slots b, C) and
// the shared prediction fp = F P (T0), pp = F P F^T + Q (T1), xp = F x + u
// (t2) (kalman_elems.hpp:151-193): E^T = pp^-1 fp, g = x - E xp,
// L = P - E fp.  Result in the slots E_k = T4, g_k = t3, L_k = T5.
template <typename S>
__device__ void smoother_elem_pred(const Step<S>& st, unsigned& err) {
  const int n = st.nx;
  WM<S> fp = st.T(0), pp = st.T(1);
  // [pp | fp] (slots T2..T3) -> [I | pp^-1 fp] = [I | E^T]
  WM<S> aug{st.T(2).p, 2 * n};
  copy(aug, pp, n, n);
  copy(WM<S>{aug.p + n, 2 * n}, fp, n, n);
  gauss_jordan(aug, n, 2 * n, false, err);
  const WM<S> et{aug.p + n, 2 * n};
  for_each(n, n, [&](int r, int c) { st.T(4)(r, c) = et(c, r); });
  gemm<true, false>(st.t(3), et, st.t(2), n, n, 1, st.b().p, 1, S(-1));
  gemm<true, false>(st.T(5), et, fp, n, n, n, st.C().p, kLd, S(-1), true);
}
// Terminal element a_T = (0, x_T, P_T) (kalman_elems.hpp:158-163) into the
// same slots.
template <typename S>
__device__ void terminal_elem(const Step<S>& st) {
  const int n = st.nx;
  fill(st.T(4), n, n, S(0), S(0));
  copy(st.t(3), st.b(), n, 1);
  copy(st.T(5), st.C(), n, n);
}
// Store the element in (T4, t3, T5) to global (AoS E, g, L) and fold it into
// the running chunk element sa = (E_a: slot A, g_a: t4, L_a: slot J).
template <typename S>
__device__ void store_and_fold(const Step<S>& st, S* out, bool first) {
  const int n = st.nx;
  const SOffs F(n);
  gstore(out + F.E, st.T(4), n, n);
  gstore(out + F.g, st.t(3), n, 1);
  gstore(out + F.L, st.T(5), n, n);
  if (first) {
    copy(st.A(), st.T(4), n, n);
    copy(st.t(4), st.t(3), n, 1);
    copy(st.J(), st.T(5), n, n);
    return;
  }
  // L_a' = E_a L_k E_a^T + L_a ; g_a' = E_a g_k + g_a ; E_a' = E_a E_k
  gemm<false, false>(st.T(2), st.A(), st.T(5), n, n, n);
  gemm<false, true>(st.J(), st.T(2), st.A(), n, n, n, st.J().p, kLd, S(1), true);
  gemm<false, false>(st.t(4), st.A(), st.t(3), n, n, 1, st.t(4).p, 1);
  gemm<false, false>(st.T(6), st.A(), st.T(4), n, n, n);
  copy(st.A(), st.T(6), n, n);
}
// Measurement update of the state (b, C) = (x, P) (kalman_seq.hpp:58-99)
template <typename S>
__device__ void kf_update(const Step<S>& st, unsigned& err) {
  const int nx = st.nx, ny = st.ny;
  WM<S> hc = st.T(2);
  WM<S> v = st.t(0);
  // [S | H P | v] (<= 16 x 33, slots T3..T4) -> [I | K^T | S^-1 v]
  const int w = ny + nx + 1;
  WM<S> aug{st.T(3).p, w};
  WM<S> kt{aug.p + ny, w}, sv{aug.p + ny + nx, w};
  gemm<false, false>(hc, st.H(), st.C(), ny, nx, nx);
  gemm<false, false>(v, st.H(), st.b(), ny, nx, 1, st.y().p, 1, S(-1));
  vadd(v, v, st.d(), ny, S(-1));
  gemm<false, true>(aug, hc, st.H(), ny, nx, ny, st.R().p, st.R().ld, S(1), true);
  copy(kt, hc, ny, nx);
  copy(sv, v, ny, 1);
  gauss_jordan(aug, ny, w, false, err);
  gemm<true, false>(st.b(), kt, v, nx, ny, 1, st.b().p, 1);
  gemm<true, false>(st.C(), kt, hc, nx, ny, nx, st.C().p, kLd, S(-1), true);
}
// shared prediction from (b, C) with F, Q, u in their slots
template <typename S>
__device__ void predict(const Step<S>& st) {
  const int n = st.nx;
  gemm<false, false>(st.T(0), st.F(), st.C(), n, n, n);
  gemm<false, true>(st.T(1), st.T(0), st.F(), n, n, n, st.Q().p, st.Q().ld, S(1), true);
  gemm<false, false>(st.t(2), st.F(), st.b(), n, n, 1, st.u().p, 1);
}

// finish: filter the chunk from the carried prefix.  SMOOTH = false writes
// the filtered stats; SMOOTH = true writes the per-step smoothing elements
// (AoS at egl + k * SS) and the chunk's smoother element (sagg + c * SS).
template <typename S, bool SMOOTH>
__global__ void __launch_bounds__(32 * kWarps)
    k_wide_finish(ModelView<S> m, long long L, long long nchunks, const S* pre,
                  const S* carry, S* mean, S* cov, S* sagg, S* egl, unsigned* err) {
  const long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= nchunks) return;
  const int nx = m.nx, ny = m.ny;
  const Step<S> st(m, nx, ny);
  unsigned e = 0;
  const long long k0 = c * L, k1 = min(k0 + L, m.t);
  const FOffs FO(nx);
  const SOffs SO(nx);
  // incoming filtered state (x, P) -> slots (b, C)
  if (c == 0) {
    gload(st.b(), m.prior_first ? m.m0 : carry, nx, 1);
    gload(st.C(), m.prior_first ? m.p0 : carry + nx, nx, nx);
    __syncwarp();
  } else if (carry == nullptr) {
    gload(st.b(), pre + (c - 1) * FO.size + FO.b, nx, 1);
    gload(st.C(), pre + (c - 1) * FO.size + FO.C, nx, nx);
    __syncwarp();
  } else {
    // carry (x) prefix(c-1), the reduced Lemma 1 with a state (A = 0) on the
    // left: M = I + P J_e, x' = A_e M^-1 (x + P eta_e) + b_e,
    // P' = A_e M^-1 P A_e^T + C_e.  The element is staged in T0..T2.
    S* el = st.T(0).p;
    for (int i = lane_id(); i < FO.size; i += 32) el[i] = pre[(c - 1) * FO.size + i];
    gload(st.b(), carry, nx, 1);
    gload(st.C(), carry + nx, nx, nx);
    __syncwarp();
    WM<S> Ae{el + FO.A, nx}, be{el + FO.b, 1}, Ce{el + FO.C, nx}, etae{el + FO.eta, 1},
        Je{el + FO.J, nx};
    // [M | I] (slots T3..T4) -> [I | M^-1]
    WM<S> aug{st.T(3).p, 2 * nx};
    WM<S> t1 = st.T(5), t2 = st.T(6);
    gemm<false, false>(aug, st.C(), Je, nx, nx, nx);
    for_each(nx, nx, [&](int i, int j) {
      aug(i, nx + j) = i == j ? S(1) : S(0);
      if (i == j) aug(i, i) += S(1);
    });
    __syncwarp();
    gauss_jordan(aug, nx, 2 * nx, true, e);
    const WM<S> Mi{aug.p + nx, 2 * nx};
    gemm<false, false>(st.t(1), st.C(), etae, nx, nx, 1, st.b().p, 1);
    gemm<false, false>(st.t(2), Mi, st.t(1), nx, nx, 1);
    gemm<false, false>(t1, Mi, st.C(), nx, nx, nx);
    gemm<false, false>(st.b(), Ae, st.t(2), nx, nx, 1, be.p, 1);
    gemm<false, false>(t2, Ae, t1, nx, nx, nx);
    gemm<false, true>(st.C(), t2, Ae, nx, nx, nx, Ce.p, nx, S(1), true);
  }
  for (long long k = k0; k < k1; ++k) {
    st.load(m, k);
    predict(st);
    if constexpr (SMOOTH) {
      if (k > k0) {  // (b, C) still hold the filtered step k-1
        smoother_elem_pred(st, e);
        store_and_fold(st, egl + (k - 1) * SO.size, k - 1 == k0);
      }
    }
    copy(st.b(), st.t(2), nx, 1);  // x = xp, P = pp
    copy(st.C(), st.T(1), nx, nx);
    kf_update(st, e);
    if constexpr (!SMOOTH) {
      gstore(mean + k * nx, st.b(), nx, 1);
      gstore(cov + k * nx * nx, st.C(), nx, nx);
      __syncwarp();
    }
  }
  if constexpr (SMOOTH) {  // element of the chunk's last step
    if (k1 - 1 == m.last_step) {
      terminal_elem(st);
    } else {
      st.load_fqu(m, k1);
      predict(st);
      smoother_elem_pred(st, e);
    }
    store_and_fold(st, egl + (k1 - 1) * SO.size, k1 - 1 == k0);
    S* o = sagg + c * SO.size;
    gstore(o + SO.E, st.A(), nx, nx);
    gstore(o + SO.g, st.t(4), nx, 1);
    gstore(o + SO.L, st.J(), nx, nx);
  }
  if (e && lane_id() == 0) atomicOr(err, e);
}

// smoother finish: backwards over the chunk from the carried suffix,
// x_s(k) = E_k x_s(k+1) + g_k, P_s(k) = E_k P_s(k+1) E_k^T + L_k.
// Slots: gs = t0, Ls = C, E_k = T0, g_k = t1, L_k = T1, W = T2, t2 tmp.
template <typename S>
__global__ void __launch_bounds__(32 * kWarps)
    k_wide_smoother_finish(ModelView<S> m, long long L, long long nchunks, const S* suf,
                           const S* carry, const S* egl, S* mean, S* cov) {
  const long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= nchunks) return;
  const int n = m.nx;
  const Step<S> st(m, n, m.ny);
  const long long k0 = c * L, k1 = min(k0 + L, m.t);
  const SOffs SO(n);
  WM<S> gs = st.t(0), Ls = st.C();
  if (c + 1 < nchunks) {
    const S* s1 = suf + (c + 1) * SO.size;
    gload(gs, s1 + SO.g, n, 1);
    gload(Ls, s1 + SO.L, n, n);
    __syncwarp();
    if (carry != nullptr) {  // (suffix of c+1) (x) carry, E of the carry = 0
      gload(st.T(0), s1 + SO.E, n, n);
      gload(st.t(1), carry, n, 1);
      gload(st.T(1), carry + n, n, n);
      __syncwarp();
      gemm<false, false>(gs, st.T(0), st.t(1), n, n, 1, gs.p, 1);
      gemm<false, false>(st.T(2), st.T(0), st.T(1), n, n, n);
      gemm<false, true>(Ls, st.T(2), st.T(0), n, n, n, Ls.p, kLd, S(1), true);
    }
  } else {
    if (carry != nullptr) {
      gload(gs, carry, n, 1);
      gload(Ls, carry + n, n, n);
    } else {  // the last step has E = 0: the incoming state is never used
      fill(gs, n, 1, S(0), S(0));
      fill(Ls, n, n, S(0), S(0));
    }
    __syncwarp();
  }
  for (long long i = k1 - 1; i >= k0; --i) {
    const S* ek = egl + i * SO.size;
    gload(st.T(0), ek + SO.E, n, n);
    gload(st.t(1), ek + SO.g, n, 1);
    gload(st.T(1), ek + SO.L, n, n);
    __syncwarp();
    gemm<false, false>(st.t(2), st.T(0), gs, n, n, 1, st.t(1).p, 1);
    copy(gs, st.t(2), n, 1);
    gemm<false, false>(st.T(2), st.T(0), Ls, n, n, n);
    gemm<false, true>(Ls, st.T(2), st.T(0), n, n, n, st.T(1).p, kLd, S(1), true);
    gstore(mean + i * n, gs, n, 1);
    gstore(cov + i * n * n, Ls, n, n);
    __syncwarp();
  }
}

// one packed element (AoS slot i of a wide buffer) -> out
template <typename S>
__global__ void k_wide_extract(const S* buf, long long i, int size, S* out) {
  for (int c = threadIdx.x; c < size; c += blockDim.x) out[c] = buf[i * size + c];
}

// padding slots [from, to) <- identity (one warp per slot)
template <class Ops>
__global__ void __launch_bounds__(128)
    k_wide_fill_identity(Ops ops, ElemBuf<typename Ops::S> b, long long from, long long to) {
  const long long i = from + (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i < to) ops.identity(b, i);
}

// ---- host dispatch -----------------------------------------------------------
inline int wide_blocks(long long warps, int per_block) {
  const long long g = (warps + per_block - 1) / per_block;
  return (int)(g < 1 ? 1 : g);
}

template <typename S>
long long wide_auto_chunk(long long T, int waves, int nm) {
  const int smem = step_smem<S>(nm);
  const int per_sm = kernel_setup(k_wide_finish<S, true>, 32 * kWarps, smem);
  const long long resident = (long long)device_sms() * (per_sm > 0 ? per_sm : 1) *
                             kWarps * (waves > 0 ? waves : 4);  // 0: default 4
  const long long L = (T + resident - 1) / resident;
  return L < 1 ? 1 : L;
}

// Level-by-level chunk scan with one warp per combine.
template <class Ops>
void wide_scan(ExactLaunch& L, const Ops& ops, typename Ops::S* buf, long long npad,
               typename Ops::S* aux1, typename Ops::S* aux2, const ScanPlan& plan, int rev) {
  using S = typename Ops::S;
  Bufs3<Ops> bufs;
  bufs.b[0] = ElemBuf<S>{buf, npad, npad, rev};
  bufs.b[1] = ElemBuf<S>{aux1, plan.cap1 ? plan.cap1 : 1, plan.cap1, rev};
  bufs.b[2] = ElemBuf<S>{aux2, plan.cap2 ? plan.cap2 : 1, plan.cap2, rev};
  const int smem = 4 * warp_bytes<S>();
  kernel_setup(k_level<Ops, 32>, 128, smem);
  for (const LevelDesc& d : plan.levels) {
    const int g = d.kind == kLvSeqChain ? 1 : (int)std::min<long long>(wide_blocks(d.count, 4),
                                                                       148LL * 16);
    k_level<Ops, 32><<<g, 128, smem, L.stream>>>(ops, bufs, d);
    L.count("chunk_scan_level_wide");
  }
}

// PKF (method 0) and PRTS (method 1) for runtime nx, ny <= 16; PTFS returns
// -1 (served by the exact path).  The decoupled look-back request (alg 6) runs
// the Ladner-Fischer plan.
template <typename S>
int wide_run(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a, S* mean, S* cov,
             void* (*alloc)(size_t, void*), void* actx) {
  if (a.method == 2 || m.nx > kMaxN || m.ny > kMaxN) return -1;
  const long long T = m.t;
  if (T == 0) return 0;
  const int nx = m.nx;
  const int nm = step_slots(m);
  long long Lc = a.chunk >= 1 ? a.chunk : wide_auto_chunk<S>(T, a.waves, nm);
  if (a.chunk < 1 && a.alg == 0 && Lc < seq_chunk_floor(T)) Lc = seq_chunk_floor(T);
  const long long nch = (T + Lc - 1) / Lc;
  const int alg = a.alg == 6 ? 3 : a.alg;
  const long long npad = alg == 0 ? nch : (long long)next_pow2(nch);
  ScanPlan plan;
  if (npad > 1) {
    plan = make_scan_plan(alg, a.sengupta_n, npad);
    if (plan.status) return plan.status;
  }
  const FOffs FO(nx);
  const SOffs SO(nx);
  const long long FS = FO.size, SS = SO.size;
  S* agg = (S*)alloc(sizeof(S) * FS * npad, actx);
  S* aux1 = (S*)alloc(sizeof(S) * FS * (plan.cap1 ? plan.cap1 : 1), actx);
  S* aux2 = (S*)alloc(sizeof(S) * FS * (plan.cap2 ? plan.cap2 : 1), actx);
  S* sagg = a.method == 1 ? (S*)alloc(sizeof(S) * SS * npad, actx) : nullptr;
  S* egl = a.method == 1 ? (S*)alloc(sizeof(S) * SS * T, actx) : nullptr;
  if (!agg || !aux1 || !aux2 || (a.method == 1 && (!sagg || !egl))) return 8;
  const int smem = step_smem<S>(nm);
  const int grid = wide_blocks(nch, kWarps);
  WideFilterOps<S> fops{L.err, nx};
  WideSmootherOps<S> sops{nx};
  // 1. reduce + scan of the filtering chunk elements
  kernel_setup(k_wide_reduce<S>, 32 * kWarps, smem);
  k_wide_reduce<S><<<grid, 32 * kWarps, smem, L.stream>>>(m, Lc, nch, agg, L.err);
  L.count("wide_filter_reduce");
  if (npad > nch) {
    k_wide_fill_identity<<<wide_blocks(npad - nch, 4), 128, 0, L.stream>>>(
        fops, ElemBuf<S>{agg, npad, npad, 0}, nch, npad);
    L.count("fill_identity");
  }
  if (npad > 1) wide_scan(L, fops, agg, npad, aux1, aux2, plan, 0);
  // 2. finish
  if (a.method == 0) {
    kernel_setup(k_wide_finish<S, false>, 32 * kWarps, smem);
    k_wide_finish<S, false><<<grid, 32 * kWarps, smem, L.stream>>>(
        m, Lc, nch, agg, nullptr, mean, cov, nullptr, nullptr, L.err);
    L.count("wide_filter_finish");
    return 0;
  }
  kernel_setup(k_wide_finish<S, true>, 32 * kWarps, smem);
  k_wide_finish<S, true><<<grid, 32 * kWarps, smem, L.stream>>>(m, Lc, nch, agg, nullptr, mean,
                                                                 cov, sagg, egl, L.err);
  L.count("wide_filter_finish_smoother_reduce");
  // 3. reverse scan of the smoothing chunk elements + smoother finish
  if (npad > nch) {
    k_wide_fill_identity<<<wide_blocks(npad - nch, 4), 128, 0, L.stream>>>(
        sops, ElemBuf<S>{sagg, npad, npad, 0}, nch, npad);
    L.count("fill_identity");
  }
  if (npad > 1) wide_scan(L, sops, sagg, npad, aux1, aux2, plan, 1);
  kernel_setup(k_wide_smoother_finish<S>, 32 * kWarps, smem);
  k_wide_smoother_finish<S><<<grid, 32 * kWarps, smem, L.stream>>>(m, Lc, nch, sagg, nullptr,
                                                                   egl, mean, cov);
  L.count("wide_smoother_finish");
  return 0;
}

}  // namespace wide
}  // namespace psk
