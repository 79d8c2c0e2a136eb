// psk_fast.cuh -- fast-path kernels (compile-time NX, NY; FP32 / FP64).
//
// Formulation: the time axis is cut into chunks of L
// consecutive steps, one chunk per thread.
//   reduce:  the thread folds its L steps into ONE scan element.  For the
//            filter this is the element of Lemma 1 (kalman_elems.hpp:53-149,
//            267-336) built by a "conditional Kalman" recursion -- the element
//            of step k composed onto the running aggregate without forming
//            the per-step element -- which costs no 4x4 LU per step.
//   scan:    the chunk elements are scanned with the selected ScanAlg
//            (psk_levels.cuh / psk_dlb.cuh) using the full Lemma-1/2
//            combines below (the register-resident associative operator).
//   finish:  the thread re-runs its chunk as a plain sequential recursion
//            starting from the carried prefix and writes the outputs.  The
//            carried filter prefix always contains a_1 (A = 0), so only its
//            (b, C) -- the filtered state -- is needed; likewise the smoother
//            suffix contains a_T (E = 0) and only (g, L) is needed.
// With L = 1 this is exactly the paper's element-per-step scan (Alg. 5-7).
#pragma once
#include "psk_common.cuh"
#include "psk_mat.cuh"
#include "psk_stage.cuh"

namespace psk {

// ---- element types --------------------------------------------------------
template <typename S, int NX>
struct FElem {  // filtering element (A, b, C, eta, J), kalman_elems.hpp:23-30
  Mat<S, NX, NX> A;
  Vec<S, NX> b;
  Mat<S, NX, NX> C;
  Vec<S, NX> eta;
  Mat<S, NX, NX> J;
};
template <typename S, int NX>
struct SElem {  // smoothing element (E, g, L), kalman_elems.hpp:32-37
  Mat<S, NX, NX> E;
  Vec<S, NX> g;
  Mat<S, NX, NX> L;
};
template <int NX>
struct FLayout {  // SoA component offsets (same packing as the oracle)
  static constexpr int A = 0, b = NX * NX, C = NX * NX + NX,
                       eta = 2 * NX * NX + NX, J = 2 * NX * NX + 2 * NX,
                       size = 3 * NX * NX + 2 * NX;
};
template <int NX>
struct SLayout {
  static constexpr int E = 0, g = NX * NX, L = NX * NX + NX,
                       size = 2 * NX * NX + NX;
};

// Per-step smoothing elements (E, g, L) written by the PRTS filter finish and
// consumed by the smoother finish (an internal buffer, so its layout is free):
// L is symmetric and only its upper triangle is kept (NX(NX+1)/2 scalars).
// Step j of chunk c lives at comp * cap ... with index (j * kSize + comp) *
// cap + c: consecutive chunks (= consecutive threads) are adjacent, so every
// access is a coalesced 32-lane transaction.
template <int NX>
struct EglLayout {
  static constexpr int E = 0, g = NX * NX, L = NX * NX + NX,
                       size = NX * NX + NX + NX * (NX + 1) / 2;
};
// (global = false: plain stores, e.g. into shared memory)
template <typename S, int NX>
__device__ __forceinline__ void egl_store(S* p, long long cap, const SElem<S, NX>& e,
                                          bool global = true) {
  using Lo = EglLayout<NX>;
  auto put = [&](int comp, S v) {
    if (global)
      __stcs(p + comp * cap, v);
    else
      p[comp * cap] = v;
  };
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) put(Lo::E + i * NX + j, e.E.a[i][j]);
#pragma unroll
  for (int i = 0; i < NX; ++i) put(Lo::g + i, e.g.a[i][0]);
  int q = Lo::L;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = i; j < NX; ++j) put(q++, e.L.a[i][j]);
}
template <typename S, int NX>
__device__ __forceinline__ SElem<S, NX> egl_load(const S* p, long long cap) {
  using Lo = EglLayout<NX>;
  SElem<S, NX> e;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = 0; j < NX; ++j) e.E.a[i][j] = __ldcs(p + (Lo::E + i * NX + j) * cap);
#pragma unroll
  for (int i = 0; i < NX; ++i) e.g.a[i][0] = __ldcs(p + (Lo::g + i) * cap);
  int q = Lo::L;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = i; j < NX; ++j) {
      const S v = __ldcs(p + (q++) * cap);
      e.L.a[i][j] = v;
      e.L.a[j][i] = v;
    }
  return e;
}

// Per-step filtered states (x, upper P) handed from the PTFS forward finish to
// the backward finish in the same chunk-interleaved layout as the smoothing
// elements (index (j * size + comp) * cap + chunk: coalesced both ways).
template <int NX>
struct StateLayout {
  static constexpr int x = 0, P = NX, size = NX + NX * (NX + 1) / 2;
};
template <typename S, int NX>
__device__ __forceinline__ void state_store(S* p, long long cap, const Vec<S, NX>& x,
                                            const Mat<S, NX, NX>& P) {
#pragma unroll
  for (int i = 0; i < NX; ++i) __stcs(p + i * cap, x.a[i][0]);
  int q = NX;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = i; j < NX; ++j) __stcs(p + (q++) * cap, P.a[i][j]);
}
template <typename S, int NX>
__device__ __forceinline__ void state_load(const S* p, long long cap, Vec<S, NX>& x,
                                           Mat<S, NX, NX>& P) {
#pragma unroll
  for (int i = 0; i < NX; ++i) x.a[i][0] = __ldcs(p + i * cap);
  int q = NX;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = i; j < NX; ++j) {
      const S v = __ldcs(p + (q++) * cap);
      P.a[i][j] = v;
      P.a[j][i] = v;
    }
}

template <typename S, int NX>
__device__ __forceinline__ FElem<S, NX> fe_load(const S* p, long long cap,
                                                long long i) {
  using Lo = FLayout<NX>;
  FElem<S, NX> e;
  e.A = load_soa<S, NX, NX>(p + Lo::A * cap + i, cap);
  e.b = load_soa<S, NX, 1>(p + Lo::b * cap + i, cap);
  e.C = load_soa<S, NX, NX>(p + Lo::C * cap + i, cap);
  e.eta = load_soa<S, NX, 1>(p + Lo::eta * cap + i, cap);
  e.J = load_soa<S, NX, NX>(p + Lo::J * cap + i, cap);
  return e;
}
template <typename S, int NX>
__device__ __forceinline__ void fe_store(S* p, long long cap, long long i,
                                         const FElem<S, NX>& e) {
  using Lo = FLayout<NX>;
  store_soa(p + Lo::A * cap + i, cap, e.A);
  store_soa(p + Lo::b * cap + i, cap, e.b);
  store_soa(p + Lo::C * cap + i, cap, e.C);
  store_soa(p + Lo::eta * cap + i, cap, e.eta);
  store_soa(p + Lo::J * cap + i, cap, e.J);
}
template <typename S, int NX>
__device__ __forceinline__ SElem<S, NX> se_load(const S* p, long long cap,
                                                long long i) {
  using Lo = SLayout<NX>;
  SElem<S, NX> e;
  e.E = load_soa<S, NX, NX>(p + Lo::E * cap + i, cap);
  e.g = load_soa<S, NX, 1>(p + Lo::g * cap + i, cap);
  e.L = load_soa<S, NX, NX>(p + Lo::L * cap + i, cap);
  return e;
}
template <typename S, int NX>
__device__ __forceinline__ void se_store(S* p, long long cap, long long i,
                                         const SElem<S, NX>& e) {
  using Lo = SLayout<NX>;
  store_soa(p + Lo::E * cap + i, cap, e.E);
  store_soa(p + Lo::g * cap + i, cap, e.g);
  store_soa(p + Lo::L * cap + i, cap, e.L);
}
template <typename S, int NX>
__device__ __forceinline__ FElem<S, NX> fe_identity() {  // (I,0,0,0,0)
  FElem<S, NX> e;
  e.A = eye<S, NX>();
  e.b = zeros<S, NX, 1>();
  e.C = zeros<S, NX, NX>();
  e.eta = zeros<S, NX, 1>();
  e.J = zeros<S, NX, NX>();
  return e;
}
template <typename S, int NX>
__device__ __forceinline__ SElem<S, NX> se_identity() {  // (I,0,0)
  SElem<S, NX> e;
  e.E = eye<S, NX>();
  e.g = zeros<S, NX, 1>();
  e.L = zeros<S, NX, NX>();
  return e;
}

// ---- Lemma 1 combine (kalman_elems.hpp:267-336), one LU --------------------
// l = earlier element (i), r = later element (j).  N = I + J_j C_i equals
// (I + C_i J_j)^T exactly because C and J are symmetric, so both solves reuse
// one factorisation (the reference factors M and N separately).
template <typename S, int NX>
__device__ __forceinline__ FElem<S, NX> filter_combine(const FElem<S, NX>& l,
                                                       const FElem<S, NX>& r,
                                                       unsigned& err) {
  FElem<S, NX> o;
  Mat<S, NX, NX> m = mul(l.C, r.J);
#pragma unroll
  for (int i = 0; i < NX; ++i) m.a[i][i] += S(1);
  const LU<S, NX> lu = lu_factor(m, err);
  {  // A' = A_j M^-1 A_i ; b' = A_j M^-1 (b_i + C_i eta_j) + b_j
    const Mat<S, NX, NX> xa = lu_solve(lu, l.A);
    o.A = mul(r.A, xa);
    const Vec<S, NX> rb = mul_add(l.C, r.eta, l.b);
    const Vec<S, NX> z = lu_solve(lu, rb);
    o.b = mul_add(r.A, z, r.b);
  }
  {  // C' = A_j M^-1 C_i A_j^T + C_j (symmetric)
    const Mat<S, NX, NX> xc = lu_solve(lu, l.C);
    const Mat<S, NX, NX> w = mul(r.A, xc);
    o.C = mul_nt_sym_add(w, r.A, r.C);
  }
  {  // eta' = A_i^T N^-1 (eta_j - J_j b_i) + eta_i
    const Vec<S, NX> w = sub_mul(r.eta, r.J, l.b);
    const Vec<S, NX> y = lu_solve_t(lu, w);
    o.eta = mul_tn_add(l.A, y, l.eta);
  }
  {  // J' = A_i^T N^-1 J_j A_i + J_i (symmetric)
    const Mat<S, NX, NX> y = lu_solve_t(lu, r.J);
    const Mat<S, NX, NX> v = mul(y, l.A);
    o.J = mul_tn_sym_add(l.A, v, l.J);
  }
  return o;
}

// ---- Lemma 2 combine (kalman_elems.hpp:396-418) -----------------------------
template <typename S, int NX>
__device__ __forceinline__ SElem<S, NX> smoother_combine(const SElem<S, NX>& l,
                                                         const SElem<S, NX>& r) {
  SElem<S, NX> o;
  o.E = mul(l.E, r.E);
  o.g = mul_add(l.E, r.g, l.g);
  const Mat<S, NX, NX> el = mul(l.E, r.L);
  o.L = mul_nt_sym_add(el, l.E, l.L);
  return o;
}

// ---- level-scan operator policies ----------------------------------------
// component-wise warp shuffle of a register matrix: y = f(x) per entry
template <typename S, int R, int C, class Shfl>
__device__ __forceinline__ void shfl_mat(Mat<S, R, C>& y, const Mat<S, R, C>& x, Shfl&& f) {
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) y.a[i][j] = f(x.a[i][j]);
}

template <typename S_, int NX>
struct FastFilterOps {
  using S = S_;
  using Elem = FElem<S, NX>;
  static constexpr int kSize = FLayout<NX>::size;
  unsigned* err;
  // register-level interface (the DLB's warp-shuffle scans, psk_dlb.cuh)
  __device__ Elem get(const ElemBuf<S>& b, long long i) const { return fe_load<S, NX>(b.p, b.cap, i); }
  __device__ void put(const ElemBuf<S>& b, long long i, const Elem& x) const {
    fe_store(b.p, b.cap, i, x);
  }
  __device__ Elem comb(const Elem& l, const Elem& r) const {
    unsigned e = 0;
    const Elem o = filter_combine(l, r, e);
    if (e) atomicOr(err, e);
    return o;
  }
  template <class Shfl>
  __device__ static Elem shfl(const Elem& x, Shfl&& f) {
    Elem y;
    shfl_mat(y.A, x.A, f);
    shfl_mat(y.b, x.b, f);
    shfl_mat(y.C, x.C, f);
    shfl_mat(y.eta, x.eta, f);
    shfl_mat(y.J, x.J, f);
    return y;
  }
  __device__ void combine(const ElemBuf<S>& d, long long di,
                          const ElemBuf<S>& l, long long li,
                          const ElemBuf<S>& r, long long ri) const {
    unsigned e = 0;
    const FElem<S, NX> a = fe_load<S, NX>(l.p, l.cap, li);
    const FElem<S, NX> b = fe_load<S, NX>(r.p, r.cap, ri);
    const FElem<S, NX> o = filter_combine(a, b, e);
    fe_store(d.p, d.cap, di, o);
    if (e) atomicOr(err, e);
  }
  __device__ void assign(const ElemBuf<S>& d, long long di,
                         const ElemBuf<S>& s, long long si) const {
    for (int c = 0; c < FLayout<NX>::size; ++c)
      d.p[c * d.cap + di] = s.p[c * s.cap + si];
  }
  __device__ void identity(const ElemBuf<S>& d, long long di) const {
    fe_store(d.p, d.cap, di, fe_identity<S, NX>());
  }
};
template <typename S_, int NX>
struct FastSmootherOps {
  using S = S_;
  using Elem = SElem<S, NX>;
  static constexpr int kSize = SLayout<NX>::size;
  unsigned* err;
  __device__ Elem get(const ElemBuf<S>& b, long long i) const { return se_load<S, NX>(b.p, b.cap, i); }
  __device__ void put(const ElemBuf<S>& b, long long i, const Elem& x) const {
    se_store(b.p, b.cap, i, x);
  }
  __device__ Elem comb(const Elem& l, const Elem& r) const { return smoother_combine(l, r); }
  template <class Shfl>
  __device__ static Elem shfl(const Elem& x, Shfl&& f) {
    Elem y;
    shfl_mat(y.E, x.E, f);
    shfl_mat(y.g, x.g, f);
    shfl_mat(y.L, x.L, f);
    return y;
  }
  __device__ void combine(const ElemBuf<S>& d, long long di,
                          const ElemBuf<S>& l, long long li,
                          const ElemBuf<S>& r, long long ri) const {
    const SElem<S, NX> a = se_load<S, NX>(l.p, l.cap, li);
    const SElem<S, NX> b = se_load<S, NX>(r.p, r.cap, ri);
    se_store(d.p, d.cap, di, smoother_combine(a, b));
  }
  __device__ void assign(const ElemBuf<S>& d, long long di,
                         const ElemBuf<S>& s, long long si) const {
    for (int c = 0; c < SLayout<NX>::size; ++c)
      d.p[c * d.cap + di] = s.p[c * s.cap + si];
  }
  __device__ void identity(const ElemBuf<S>& d, long long di) const {
    se_store(d.p, d.cap, di, se_identity<S, NX>());
  }
};

// ---- per-step building blocks ---------------------------------------------
template <typename S, int NX, int NY>
struct Meas {
  Mat<S, NY, NX> H;
  Vec<S, NY> d;
  Mat<S, NY, NY> R;
  Vec<S, NY> y;
};
template <typename S, int NX, int NY>
__device__ __forceinline__ Meas<S, NX, NY> load_meas(const ModelView<S>& m,
                                                     long long k) {
  Meas<S, NX, NY> z;
  z.H = load<S, NY, NX>(m.H(k));
  z.d = load<S, NY, 1>(m.D(k));
  z.R = load<S, NY, NY>(m.R(k));
  z.y = load<S, NY, 1>(m.Y(k));
  return z;
}

// Kalman update of a state (kalman_seq.hpp:58-99): (x, P)_{k|k-1} -> k|k
template <typename S, int NX, int NY>
__device__ __forceinline__ void kf_update(Vec<S, NX>& x, Mat<S, NX, NX>& P,
                                          const Meas<S, NX, NY>& z,
                                          unsigned& err) {
  const Mat<S, NY, NX> hp = mul(z.H, P);
  const Mat<S, NY, NY> s = mul_nt_sym_add(hp, z.H, z.R);
  const Chol<S, NY> ch = cholesky(s, err);
  const Mat<S, NY, NX> kt = chol_solve(ch, hp);  // K^T
  Vec<S, NY> v = sub_mul(z.y, z.H, x);
  v = sub(v, z.d);
  x = mul_tn_add(kt, v, x);
  // P - K H P, symmetric
  Mat<S, NX, NX> o;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = i; j < NX; ++j) {
      S acc = P.a[i][j];
#pragma unroll
      for (int k = 0; k < NY; ++k) acc = sfma(-kt.a[k][i], hp.a[k][j], acc);
      o.a[i][j] = acc;
      o.a[j][i] = acc;
    }
  P = o;
}

// Conditional update of a filter aggregate: the predicted conditional
// (A, b, C) of x_k given the chunk-start state is updated with y_k and the
// likelihood information (eta, J) of the chunk-start state is accumulated.
// For a single step starting from the identity this is exactly
// make_filter_element (kalman_elems.hpp:97-147): A = F - KHF, b = u + Kv,
// C = Q - KHQ, eta = (HF)^T S^-1 v, J = (HF)^T S^-1 HF.
template <typename S, int NX, int NY>
__device__ __forceinline__ void cond_update(FElem<S, NX>& e,
                                            const Meas<S, NX, NY>& z,
                                            unsigned& err) {
  const Mat<S, NY, NX> hc = mul(z.H, e.C);
  const Mat<S, NY, NY> s = mul_nt_sym_add(hc, z.H, z.R);
  const Chol<S, NY> ch = cholesky(s, err);
  const Mat<S, NY, NX> kt = chol_solve(ch, hc);  // K^T
  Vec<S, NY> v = sub_mul(z.y, z.H, e.b);
  v = sub(v, z.d);
  const Mat<S, NY, NX> ha = mul(z.H, e.A);
  const Mat<S, NY, NX> w = chol_solve(ch, ha);   // S^-1 H A
  const Vec<S, NY> sv = chol_solve(ch, v);        // S^-1 v
  e.eta = mul_tn_add(ha, sv, e.eta);
  e.J = mul_tn_sym_add(ha, w, e.J);
  e.A = sub_mul_tn(e.A, kt, ha);
  e.b = mul_tn_add(kt, v, e.b);
  Mat<S, NX, NX> o;
#pragma unroll
  for (int i = 0; i < NX; ++i)
#pragma unroll
    for (int j = i; j < NX; ++j) {
      S acc = e.C.a[i][j];
#pragma unroll
      for (int k = 0; k < NY; ++k) acc = sfma(-kt.a[k][i], hc.a[k][j], acc);
      o.a[i][j] = acc;
      o.a[j][i] = acc;
    }
  e.C = o;
}

template <typename S, int NX>
__device__ __forceinline__ void store_state(S* mean, S* cov, long long k,
                                            const Vec<S, NX>& x,
                                            const Mat<S, NX, NX>& P) {
  store(mean + k * NX, x);
  store(cov + k * NX * NX, P);
}
// Reduced Lemma-1 combine of a filtered state (an element with A = 0,
// b = x, C = P) with an element e:  M = I + P J_e,
// x' = A_e M^-1 (x + P eta_e) + b_e,  P' = A_e M^-1 P A_e^T + C_e.
template <typename S, int NX>
__device__ __forceinline__ void filter_apply(Vec<S, NX>& x, Mat<S, NX, NX>& P,
                                             const FElem<S, NX>& e,
                                             unsigned& err) {
  Mat<S, NX, NX> m = mul(P, e.J);
#pragma unroll
  for (int i = 0; i < NX; ++i) m.a[i][i] += S(1);
  const LU<S, NX> lu = lu_factor(m, err);
  const Vec<S, NX> rb = mul_add(P, e.eta, x);
  const Vec<S, NX> z = lu_solve(lu, rb);
  const Mat<S, NX, NX> xc = lu_solve(lu, P);
  x = mul_add(e.A, z, e.b);
  const Mat<S, NX, NX> w = mul(e.A, xc);
  P = mul_nt_sym_add(w, e.A, e.C);
}

// ============================================================================
// Staged per-step kernels.  Each thread owns one chunk of consecutive steps;
// the CTA's step j+1 is fetched into shared memory by TMA (psk_stage.cuh)
// while step j is computed, double-buffered.  At 255 registers per FP64
// thread only 8 warps fit per SM -- far too few to hide HBM latency with
// plain loads (profiles/r01_v0: long-scoreboard stalls dominated); the stage
// keeps a whole step of the CTA in flight instead.
// ============================================================================

// This thread's view of one step: the TMA stage, or global memory for a
// broadcast field and for the ragged tail chunk (which the tensor maps --
// full chunks only -- do not cover).
template <typename S, int NX, int NY>
struct FilterStage {
  using In = FilterTma<S, NX, NY>;
  const unsigned char* st;
  int t;
  bool direct;
  const ModelView<S>* m;
  long long k;
  unsigned unstaged;  // bit f: field f is read from global memory
  unsigned g2, g4;    // bit f: field f packs 2 / 4 steps per staged row
  int j;              // walk position (k - chunk start)
  __device__ __forceinline__ bool glob(int f) const { return direct || ((unstaged >> f) & 1u); }
  // byte offset of step k's block in a grouped row of field f (block bytes
  // b; chunk starts are row-aligned): branch-free
  __device__ __forceinline__ int sub(int f, int b) const {
    const int mask = (int)((g2 >> f) & 1u) | (int)(((g4 >> f) & 1u) * 3u);
    return (j & mask) * b;
  }
  __device__ __forceinline__ Mat<S, NX, NX> F() const {
    return glob(0) ? load<S, NX, NX>(m->F(k))
                   : tma_get<typename In::F, S, NX, NX>(st, t, sub(0, In::F::bytes));
  }
  __device__ __forceinline__ Vec<S, NX> u() const {
    return glob(1) ? load<S, NX, 1>(m->U(k))
                   : tma_get<typename In::u, S, NX, 1>(st, t, sub(1, In::u::bytes));
  }
  __device__ __forceinline__ Mat<S, NX, NX> Q() const {
    return glob(2) ? load<S, NX, NX>(m->Q(k))
                   : tma_get<typename In::Q, S, NX, NX>(st, t, sub(2, In::Q::bytes));
  }
  __device__ __forceinline__ Meas<S, NX, NY> meas() const {
    Meas<S, NX, NY> z;
    z.H = glob(3) ? load<S, NY, NX>(m->H(k))
                  : tma_get<typename In::H, S, NY, NX>(st, t, sub(3, In::H::bytes));
    z.d = glob(4) ? load<S, NY, 1>(m->D(k))
                  : tma_get<typename In::d, S, NY, 1>(st, t, sub(4, In::d::bytes));
    z.R = glob(5) ? load<S, NY, NY>(m->R(k))
                  : tma_get<typename In::R, S, NY, NY>(st, t, sub(5, In::R::bytes));
    z.y = glob(6) ? load<S, NY, 1>(m->Y(k))
                  : tma_get<typename In::y, S, NY, 1>(st, t, sub(6, In::y::bytes));
    return z;
  }
};

// Multi-buffered TMA walk over this thread's chunk c = steps [k0, k1)
// (NS stages: step k's inputs are consumed while the next NS - 1 steps are in
// flight; dynamic shared memory FilterTma::smem_n(NS)).  body(k, stage) sees step k's inputs.  The
// walk is CTA-uniform (every thread of the CTA must call it: block barriers),
// of length min(L, T - first step of the CTA).  `nfull` = number of complete
// chunks (the extent of the tensor maps).
struct NoPost {
  __device__ void operator()(unsigned char*, long long) const {}
};
// `post(stage, j)` runs on thread 0 of a TMA CTA once the CTA has finished
// walk position j (after its block barrier), before the stage is refilled:
// the body may leave results in the consumed stage for a TMA store.
template <typename S, int NX, int NY, int NS = 2, class Body, class Post = NoPost>
__device__ __forceinline__ void staged_walk(unsigned char* smem_raw, const StageMaps& maps,
                                            const ModelView<S>& m, long long L, long long nfull,
                                            long long k0, long long k1, Body&& body,
                                            Post post = Post{}) {
  using In = FilterTma<S, NX, NY>;
  using St = FilterStage<S, NX, NY>;
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + NS * In::stage);
  const int t = threadIdx.x;
  const long long cta0 = (long long)blockIdx.x * kStageNT;  // first chunk of the CTA
  const bool tma = cta0 < nfull;                            // CTA-uniform
  const long long jn = min(L, m.t - cta0 * L);
  const bool direct = !tma || cta0 + t >= nfull;
  unsigned unstaged = 0, g2 = 0, g4 = 0;  // per-field flags, in registers
#pragma unroll
  for (int f = 0; f < 7; ++f) {
    unstaged |= (maps.use[f] ? 0u : 1u) << f;
    g2 |= (maps.grp[f] == 2 ? 1u : 0u) << f;
    g4 |= (maps.grp[f] == 4 ? 1u : 0u) << f;
  }
  // row of walk position j in field f's box: j / grp, grp in {1, 2, 4} -- a
  // shift (a 64-bit division here was a ~100-instruction call per field per
  // step on the issuing thread, which the whole CTA then waited for at the
  // step barrier)
  auto grp_shift = [&](int f) { return (int)((g2 >> f) & 1u) + 2 * (int)((g4 >> f) & 1u); };
  auto issue = [&](int s, long long j) {
    fence_proxy_async();  // generic reads of this stage (last use) before the refill
    mbar_expect_tx(&bars[s], maps.tx);
#pragma unroll
    for (int f = 0; f < 7; ++f)
      if (maps.use[f])
        tma_load_3d(sm + s * In::stage + In::off(f), &maps.m[f], 0, (int)j >> grp_shift(f),
                    (int)cta0, &bars[s]);
  };
  if (tma && t == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
    mbar_init_fence();
    for (int i = 0; i < NS - 1 && i < jn; ++i) issue(i, i);
  }
  __syncthreads();
  int s = 0;           // stage of position j
  unsigned phase = 0;  // its mbarrier phase
  for (long long j = 0; j < jn; ++j) {
    // refill the stage consumed at j - 1 (all threads passed the barrier)
    if (tma && t == 0) {
      const int sp = s == 0 ? NS - 1 : s - 1;
      if (j > 0) post(sm + sp * In::stage, j - 1);
      if (j + NS - 1 < jn) issue(sp, j + NS - 1);
    }
    if (tma) mbar_wait(&bars[s], phase);
    if (k0 + j < k1) body(k0 + j, St{sm + s * In::stage, t, direct, &m, k0 + j, unstaged, g2, g4, (int)j});
    __syncthreads();  // stage s is refilled by the next iteration's issue
    if (++s == NS) {
      s = 0;
      phase ^= 1u;
    }
  }
  if (tma && t == 0 && jn > 0) post(sm + (s == 0 ? NS - 1 : s - 1) * In::stage, jn - 1);
}

// The same multi-buffered TMA walk, backwards: positions j = jn-1 .. 0 of
// the chunk (body(k0 + j, stage) for the thread's positions inside [k0, k1);
// `valid` positions are those < m.t, the others see no data).  `jn` is the
// CTA-uniform walk length chosen by the caller.
template <typename S, int NX, int NY, int NS = 2, class Body>
__device__ __forceinline__ void staged_walk_rev(unsigned char* smem_raw, const StageMaps& maps,
                                                const ModelView<S>& m, long long L,
                                                long long nfull, long long jn, long long k0,
                                                long long k1, Body&& body) {
  using In = FilterTma<S, NX, NY>;
  using St = FilterStage<S, NX, NY>;
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + NS * In::stage);
  const int t = threadIdx.x;
  const long long cta0 = (long long)blockIdx.x * kStageNT;
  const bool tma = cta0 < nfull;
  const bool direct = !tma || cta0 + t >= nfull;
  unsigned unstaged = 0, g2 = 0, g4 = 0;  // per-field flags, in registers
#pragma unroll
  for (int f = 0; f < 7; ++f) {
    unstaged |= (maps.use[f] ? 0u : 1u) << f;
    g2 |= (maps.grp[f] == 2 ? 1u : 0u) << f;
    g4 |= (maps.grp[f] == 4 ? 1u : 0u) << f;
  }
  // positions >= the m-length of the CTA's first chunk carry no data; the
  // i-th fetch is position jd - 1 - i
  const long long jd = min(jn, max(0LL, m.t - cta0 * L));
  auto grp_shift = [&](int f) { return (int)((g2 >> f) & 1u) + 2 * (int)((g4 >> f) & 1u); };
  auto issue = [&](int s, long long j) {
    fence_proxy_async();
    mbar_expect_tx(&bars[s], maps.tx);
#pragma unroll
    for (int f = 0; f < 7; ++f)
      if (maps.use[f])
        tma_load_3d(sm + s * In::stage + In::off(f), &maps.m[f], 0, (int)j >> grp_shift(f),
                    (int)cta0, &bars[s]);
  };
  if (tma && t == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
    mbar_init_fence();
    for (int i = 0; i < NS - 1 && i < jd; ++i) issue(i, jd - 1 - i);
  }
  __syncthreads();
  int s = 0;  // stage of the next fetch consumed
  unsigned phase = 0;
  for (long long j = jn - 1; j >= 0; --j) {
    const bool data = j < jd;
    if (data) {
      if (tma && t == 0 && j - (NS - 1) >= 0) issue(s == 0 ? NS - 1 : s - 1, j - (NS - 1));
      if (tma) mbar_wait(&bars[s], phase);
    }
    const long long k = k0 + j;
    if (k < k1) body(k, k < m.t, St{sm + s * In::stage, t, direct, &m, k, unstaged, g2, g4, (int)j});
    __syncthreads();
    if (data && ++s == NS) {
      s = 0;
      phase ^= 1u;
    }
  }
}

// Smoothing element of step i from the filtered (x, P)_i and the transition
// (F, Q, u)_{i+1} passed in registers (kalman_elems.hpp:151-193).
template <typename S, int NX>
__device__ __forceinline__ SElem<S, NX> smoother_elem(const Vec<S, NX>& x,
                                                      const Mat<S, NX, NX>& P,
                                                      const Mat<S, NX, NX>& F,
                                                      const Mat<S, NX, NX>& Q,
                                                      const Vec<S, NX>& u, unsigned& err) {
  SElem<S, NX> e;
  const Mat<S, NX, NX> fp = mul(F, P);
  const Mat<S, NX, NX> pp = mul_nt_sym_add(fp, F, Q);
  const Chol<S, NX> ch = cholesky(pp, err);
  const Mat<S, NX, NX> et = chol_solve(ch, fp);  // E^T
  e.E = trans(et);
  const Vec<S, NX> fx = mul_add(F, x, u);
  e.g = sub_mul(x, e.E, fx);
  Mat<S, NX, NX> o;
#pragma unroll
  for (int a = 0; a < NX; ++a)
#pragma unroll
    for (int b = a; b < NX; ++b) {
      S acc = P.a[a][b];
#pragma unroll
      for (int k = 0; k < NX; ++k) acc = sfma(-et.a[k][a], fp.a[k][b], acc);
      o.a[a][b] = acc;
      o.a[b][a] = acc;
    }
  e.L = o;
  return e;
}
template <typename S, int NX>
__device__ __forceinline__ SElem<S, NX> terminal_elem(const Vec<S, NX>& x,
                                                      const Mat<S, NX, NX>& P) {
  SElem<S, NX> e;  // a_T = (0, x_T, P_T), kalman_elems.hpp:158-163
  e.E = zeros<S, NX, NX>();
  e.g = x;
  e.L = P;
  return e;
}

// reduce: chunk c = steps [c L, min(c L + L, T)) -> one filtering element
template <typename S, int NX, int NY>
__global__ void __launch_bounds__(kStageNT, sizeof(S) == 8 ? 2 : 3)
    k_filter_reduce(ModelView<S> m, const __grid_constant__ StageMaps maps, long long L,
                    long long nchunks, long long nfull, S* agg, long long cap, ChunkOrder ord,
                    unsigned* err) {
  extern __shared__ __align__(1024) unsigned char fsm[];
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = c < nchunks;  // idle threads stay for the block barriers
  unsigned e = 0;
  const long long k0 = c * L;
  const long long k1 = min(k0 + L, m.t);
  using St = FilterStage<S, NX, NY>;
  // Every step is composed onto the running element by the conditional
  // Kalman recursion.  From the identity (I, 0, 0, 0, 0) the first step gives
  // exactly make_filter_element (kalman_elems.hpp:97-147); the chunk holding
  // step 1 starts from the prior in state form (A = 0, b = m0, C = P0), which
  // absorbs it as a_1 does (kalman_elems.hpp:68-96) -- A, eta and J then stay
  // 0 and the element is the filtered state itself.
  FElem<S, NX> a = fe_identity<S, NX>();
  if (live && k0 == 0 && m.prior_first) {
    a.A = zeros<S, NX, NX>();
    a.b = load<S, NX, 1>(m.m0);
    a.C = load<S, NX, NX>(m.p0);
  }
  staged_walk<S, NX, NY>(fsm, maps, m, L, nfull, k0, k1, [&](long long, const St& in) {
    // predict the conditional: (F A, F b + u, F C F^T + Q), then update
    const Mat<S, NX, NX> F = in.F();
    a.A = mul(F, a.A);
    a.b = mul_add(F, a.b, in.u());
    const Mat<S, NX, NX> fc = mul(F, a.C);
    a.C = mul_nt_sym_add(fc, F, in.Q());
    cond_update(a, in.meas(), e);
  });
  if (live) fe_store(agg, cap, ord.at(c), a);
  if (e) atomicOr(err, e);
}

// Incoming filtered state of chunk c: the inclusive prefix of chunk c-1 (or
// the prior).  In a time-sharded run `carry` holds the filtered state before
// the shard and the incoming state of chunk c > 0 is carry (x) prefix(c-1),
// the reduced Lemma-1 combine of a state (A = 0) with an element.
template <typename S, int NX>
__device__ __forceinline__ void filter_incoming(const ModelView<S>& m, long long c,
                                                const S* pre, long long pre_cap,
                                                ChunkOrder pord, const S* carry,
                                                Vec<S, NX>& x, Mat<S, NX, NX>& P,
                                                unsigned& e) {
  if (c == 0) {
    if (m.prior_first) {
      x = load<S, NX, 1>(m.m0);
      P = load<S, NX, NX>(m.p0);
    } else {
      x = load<S, NX, 1>(carry);
      P = load<S, NX, NX>(carry + NX);
    }
  } else if (carry == nullptr) {
    const long long q = pord.at(c - 1);
    x = load_soa<S, NX, 1>(pre + FLayout<NX>::b * pre_cap + q, pre_cap);
    P = load_soa<S, NX, NX>(pre + FLayout<NX>::C * pre_cap + q, pre_cap);
  } else {
    x = load<S, NX, 1>(carry);
    P = load<S, NX, NX>(carry + NX);
    filter_apply(x, P, fe_load<S, NX>(pre, pre_cap, pord.at(c - 1)), e);
  }
}

// Smoothing element of step k-1 from its filtered (x, P) and the prediction
// to step k that the filter computes anyway (kalman_elems.hpp:151-193 with
// FP = F P, PP = F P F^T + Q and F x + u shared with kf_predict):
// E^T = PP^-1 FP (Cholesky), g = x - E (F x + u), L = P - E FP (symmetric).
template <typename S, int NX>
__device__ __forceinline__ SElem<S, NX> smoother_elem_pred(const Vec<S, NX>& x,
                                                           const Mat<S, NX, NX>& P,
                                                           const Mat<S, NX, NX>& fp,
                                                           const Mat<S, NX, NX>& pp,
                                                           const Vec<S, NX>& xp, unsigned& err) {
  SElem<S, NX> e;
  const Chol<S, NX> ch = cholesky(pp, err);
  const Mat<S, NX, NX> et = chol_solve(ch, fp);  // E^T
  e.E = trans(et);
  e.g = sub_mul(x, e.E, xp);
#pragma unroll
  for (int a = 0; a < NX; ++a)
#pragma unroll
    for (int b = a; b < NX; ++b) {
      S acc = P.a[a][b];
#pragma unroll
      for (int k = 0; k < NX; ++k) acc = sfma(-et.a[k][a], fp.a[k][b], acc);
      e.L.a[a][b] = acc;
      e.L.a[b][a] = acc;
    }
  return e;
}

// finish: sequential Kalman filter over the chunk from the carried prefix.
// SMOOTH = false: writes the filtered stats -- to mean/cov (PKF), or, when
// `egl` is non-null (PTFS), coalesced to the chunk-interleaved state scratch
// the backward finish reads (StateLayout).  SMOOTH = true
// (PRTS): the caller needs the smoothed stats only, so the pass writes the
// per-step smoothing elements e_k instead and folds the chunk's smoothing
// element e_{k0} (x) ... (x) e_{k1-1} into `sagg` (Lemma 2 is associative,
// so the chunk element is built forwards).  e_{k-1} needs the filtered state
// of step k-1 and the prediction to step k, which the filter computes for
// step k anyway.  The step body is branch-free (one basic block: the
// scheduler overlaps the filter, smoothing-element and fold chains); at the
// first step of a chunk the element computed from the incoming state belongs
// to the previous chunk and is replaced by the identity.
template <typename S, int NX, int NY, bool SMOOTH>
__global__ void __launch_bounds__(kStageNT, FilterTma<S, NX, NY>::finish_ctas)
    k_filter_finish(ModelView<S> m, const __grid_constant__ StageMaps maps, long long L,
                    long long nchunks, long long nfull, const S* pre, long long pre_cap,
                    ChunkOrder pord, const S* carry, S* mean, S* cov, S* sagg,
                    long long scap, ChunkOrder sord, S* egl, long long ecap, unsigned* err,
                    const __grid_constant__ EglStore em) {
  extern __shared__ __align__(1024) unsigned char fsm[];
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = c < nchunks;  // idle threads stay for the block barriers
  unsigned e = 0;
  const long long k0 = c * L;
  const long long k1 = min(k0 + L, m.t);
  constexpr int ES = EglLayout<NX>::size;
  using St = FilterStage<S, NX, NY>;
  Vec<S, NX> x = zeros<S, NX, 1>();
  Mat<S, NX, NX> P = zeros<S, NX, NX>();
  if (live) filter_incoming<S, NX>(m, c, pre, pre_cap, pord, carry, x, P, e);
  SElem<S, NX> sa = se_identity<S, NX>();
  // PRTS: in CTAs whose 128 chunks are all complete, step k's element e_{k-1}
  // goes to the consumed input stage (its F / u / Q boxes, read at the start
  // of the step) and leaves by one TMA store per walk position, instead of
  // 30 scattered 8-byte stores per thread
  const bool egl_tma = SMOOTH && em.use && ((long long)blockIdx.x + 1) * kStageNT <= nfull;
  auto post = [&](unsigned char* st, long long j) {
    if (egl_tma && j >= 1) {
      tma_store_2d(&em.map, (int)(blockIdx.x * kStageNT), (int)((j - 1) * ES), st);
      bulk_commit();
      bulk_wait_read<0>();  // the stage is refilled next
    }
  };
  staged_walk<S, NX, NY, FilterTma<S, NX, NY>::finish_stages>(
      fsm, maps, m, L, nfull, k0, k1, [&](long long k, const St& in) {
    const Mat<S, NX, NX> F = in.F();
    const Vec<S, NX> xp = mul_add(F, x, in.u());
    const Mat<S, NX, NX> fp = mul(F, P);
    const Mat<S, NX, NX> pp = mul_nt_sym_add(fp, F, in.Q());
    if constexpr (SMOOTH) {
      // (x, P) still hold the filtered step k-1
      unsigned es = 0;
      const SElem<S, NX> ek = smoother_elem_pred(x, P, fp, pp, xp, es);
      const bool keep = k > k0;
      e |= keep ? es : 0u;
      const SElem<S, NX> id = se_identity<S, NX>();
      SElem<S, NX> eu;
#pragma unroll
      for (int i = 0; i < NX; ++i) {
        eu.g.a[i][0] = keep ? ek.g.a[i][0] : id.g.a[i][0];
#pragma unroll
        for (int j = 0; j < NX; ++j) {
          eu.E.a[i][j] = keep ? ek.E.a[i][j] : id.E.a[i][j];
          eu.L.a[i][j] = keep ? ek.L.a[i][j] : id.L.a[i][j];
        }
      }
      sa = smoother_combine(sa, eu);
      if (egl_tma) {
        if (keep) {  // CTA-uniform (k - k0 is the walk position)
          // every thread's F / u / Q rows are read before any thread writes
          // over them (the element rows span all chunks' input rows)
          __syncthreads();
          S* es = reinterpret_cast<S*>(const_cast<unsigned char*>(in.st));
          egl_store(es + threadIdx.x, (long long)kStageNT, ek, false);
          fence_proxy_async();  // generic writes -> the async proxy (TMA store)
        }
      } else if (keep) {
        egl_store(egl + (k - 1 - k0) * ES * ecap + c, ecap, ek);
      }
    }
    x = xp;
    P = pp;
    kf_update(x, P, in.meas(), e);
    if constexpr (!SMOOTH) {
      if (egl == nullptr)
        store_state(mean, cov, k, x, P);
      else
        state_store(egl + (k - k0) * StateLayout<NX>::size * ecap + c, ecap, x, P);
    }
  }, post);
  if constexpr (SMOOTH) {
    if (egl_tma && threadIdx.x == 0) bulk_wait<0>();
    if (live) {  // element of the chunk's last step
      SElem<S, NX> ek;
      if (k1 - 1 == m.last_step)
        ek = terminal_elem(x, P);
      else
        ek = smoother_elem(x, P, load<S, NX, NX>(m.F(k1)), load<S, NX, NX>(m.Q(k1)),
                           load<S, NX, 1>(m.U(k1)), e);
      egl_store(egl + (k1 - 1 - k0) * ES * ecap + c, ecap, ek);
      sa = smoother_combine(sa, ek);
      se_store(sagg, scap, sord.at(c), sa);
    }
  }
  if (e) atomicOr(err, e);
}

// ============================================================================
// RTS smoother kernels (reverse direction)
// ============================================================================

// finish: sequential RTS over the chunk from the carried suffix (the
// inclusive reversed prefix of chunk c+1 = smoothed state at step k1), driven
// by the per-step smoothing elements of the filter finish:
// x_s(k) = E_k x_s(k+1) + g_k, P_s(k) = E_k P_s(k+1) E_k^T + L_k (Lemma 2
// with a state on the right).  In a time-sharded run `carry` holds the
// smoothed state after the shard (fold of the successor shards' elements,
// E = 0): the incoming state of chunk c < nchunks-1 is then
// (local suffix of chunk c+1) (x) carry.
//
// Each warp walks its 32 chunks backwards in lock-step: the elements of step
// j-1 arrive by TMA while step j is computed, and the smoothed rows of step j
// leave by TMA store (SmoothTma, psk_stage.cuh); rows the tensor maps do not
// cover (the ragged tail chunk, rows that are not whole 16-byte units) are
// stored directly.
constexpr int kSmoothNT = 64;  // 2 warps per CTA

template <typename S, int NX>
__global__ void __launch_bounds__(kSmoothNT)
    k_smoother_finish(long long t, long long L, long long nchunks, long long nfull,
                      const S* suf, long long suf_cap, ChunkOrder sord, const S* carry,
                      const __grid_constant__ SmoothMaps maps, long long ecap, S* mean, S* cov) {
  using Tm = SmoothTma<S, NX>;
  constexpr int ES = Tm::ES;
  extern __shared__ __align__(1024) unsigned char ssm_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      ((reinterpret_cast<uintptr_t>(ssm_raw) + 1023) & ~uintptr_t(1023)) + (size_t)w * Tm::warp);
  constexpr int ENS = Tm::egl_nstage;
  unsigned char* egl_st = sm;                                   // ENS x egl_stage
  unsigned char* mean_st = sm + ENS * Tm::egl_stage;            // 2 x mean_stage
  unsigned char* cov_st = mean_st + 2 * Tm::mean_stage;         // 2 x cov_stage
  uint64_t* bars = reinterpret_cast<uint64_t*>(cov_st + 2 * Tm::cov_stage);
  const long long cw0 = (long long)blockIdx.x * kSmoothNT + w * 32;  // first chunk of the warp
  if (cw0 >= nchunks) return;  // warp-uniform (no block barriers below)
  const long long c = cw0 + lane;
  const bool live = c < nchunks;
  const long long k0 = c * L;
  const long long k1 = min(k0 + L, t);
  const long long jn = min(L, t - cw0 * L);  // warp-uniform walk length
  const bool tstore = maps.store && cw0 < nfull;
  const bool direct_out = !tstore || c >= nfull;

  Vec<S, NX> gs = zeros<S, NX, 1>();
  Mat<S, NX, NX> Ls = zeros<S, NX, NX>();
  if (live && c + 1 < nchunks) {
    const long long q = sord.at(c + 1);
    gs = load_soa<S, NX, 1>(suf + SLayout<NX>::g * suf_cap + q, suf_cap);
    Ls = load_soa<S, NX, NX>(suf + SLayout<NX>::L * suf_cap + q, suf_cap);
    if (carry != nullptr) {
      const Mat<S, NX, NX> E = load_soa<S, NX, NX>(suf + SLayout<NX>::E * suf_cap + q, suf_cap);
      const Vec<S, NX> cg = load<S, NX, 1>(carry);
      const Mat<S, NX, NX> cl = load<S, NX, NX>(carry + NX);
      gs = mul_add(E, cg, gs);
      const Mat<S, NX, NX> el = mul(E, cl);
      Ls = mul_nt_sym_add(el, E, Ls);
    }
  } else if (live && carry != nullptr) {
    gs = load<S, NX, 1>(carry);
    Ls = load<S, NX, NX>(carry + NX);
  }
  // the series' last step has E = 0 (terminal element), so the zero state
  // entering the last chunk of an unsharded run is never used
  auto issue = [&](int st, long long j) {
    fence_proxy_async();
    mbar_expect_tx(&bars[st], (unsigned)Tm::egl_box);
    tma_load_2d(egl_st + st * Tm::egl_stage, &maps.egl, (int)cw0, (int)(j * ES), &bars[st]);
  };
  // the i-th fetch is position jn - 1 - i, into stage i mod ENS
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < ENS; ++i) mbar_init(&bars[i], 1);
    mbar_init_fence();
    for (int i = 0; i < ENS - 1 && i < jn; ++i) issue(i, jn - 1 - i);
  }
  __syncwarp();
  int es = 0;  // element stage of position j
  unsigned ephase = 0;
  for (long long j = jn - 1; j >= 0; --j) {
    const int st = (int)(j & 1);  // output stage
    if (lane == 0 && j - (ENS - 1) >= 0) issue(es == 0 ? ENS - 1 : es - 1, j - (ENS - 1));
    mbar_wait(&bars[es], ephase);
    const S* el = reinterpret_cast<const S*>(egl_st + es * Tm::egl_stage);
    const bool act = live && k0 + j < k1;
    if (act) {
      SElem<S, NX> ei;
      using Lo = EglLayout<NX>;
#pragma unroll
      for (int i = 0; i < NX; ++i)
#pragma unroll
        for (int q = 0; q < NX; ++q) ei.E.a[i][q] = el[(Lo::E + i * NX + q) * 32 + lane];
#pragma unroll
      for (int i = 0; i < NX; ++i) ei.g.a[i][0] = el[(Lo::g + i) * 32 + lane];
      int q = Lo::L;
#pragma unroll
      for (int i = 0; i < NX; ++i)
#pragma unroll
        for (int p = i; p < NX; ++p) {
          const S v = el[(q++) * 32 + lane];
          ei.L.a[i][p] = v;
          ei.L.a[p][i] = v;
        }
      gs = mul_add(ei.E, gs, ei.g);
      const Mat<S, NX, NX> eL = mul(ei.E, Ls);
      Ls = mul_nt_sym_add(eL, ei.E, ei.L);
    }
    if constexpr (Tm::Mean::bytes % 16 == 0 && Tm::Cov::bytes % 16 == 0) {
      if (tstore) {
        // the store issued from this stage two steps ago has left it
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        unsigned char* ms = mean_st + st * Tm::mean_stage;
        unsigned char* cs = cov_st + st * Tm::cov_stage;
        tma_put<typename Tm::Mean>(ms, lane, gs);
        tma_put<typename Tm::Cov>(cs, lane, Ls);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&maps.mean, 0, (int)j, (int)cw0, ms);
          tma_store_3d(&maps.cov, 0, (int)j, (int)cw0, cs);
          bulk_commit();
        }
      }
    }
    if (act && direct_out) store_state(mean, cov, k0 + j, gs, Ls);
    __syncwarp();  // stage es of the elements is refilled next iteration
    if (++es == ENS) {
      es = 0;
      ephase ^= 1u;
    }
  }
  if (lane == 0) bulk_wait<0>();
}

// ============================================================================
// Two-filter smoother: backward (shifted) filter + combination (K8)
// ============================================================================

// finish: backward information recursion (eta, J) <- a (x) (eta, J) over the
// chunk's slots, walking backwards, fused with tf_combine (kalman_seq.hpp:
// 236-260) against the filtered states of the forward finish (state scratch),
// writing the smoothed stats to mean/cov.  Slot i holds a_{i+2} (1-based; the element of 0-based
// step i+1) or the identity (build_shifted_filter_elems, kalman_par.hpp:
// 63-89); `ms` is the model shifted by one step (ms step i = m step i+1,
// ms.t = T - 1), staged by TMA like the forward passes.
// (eta, J) <- the eta / J rows of a (x) (., ., ., eta, J) (Lemma 1,
// kalman_elems.hpp:267-336: they depend on the right operand through its
// (eta, J) alone): N = I + J C_a, eta' = A_a^T N^-1 (eta - J b_a) + eta_a,
// J' = A_a^T N^-1 J A_a + J_a
template <typename S, int NX>
__device__ __forceinline__ void bwd_info_apply(const FElem<S, NX>& a, Vec<S, NX>& eta,
                                               Mat<S, NX, NX>& J, unsigned& e) {
  Mat<S, NX, NX> nm = mul(J, a.C);
#pragma unroll
  for (int q = 0; q < NX; ++q) nm.a[q][q] += S(1);
  const LU<S, NX> lu = lu_factor(nm, e);
  const Vec<S, NX> w = sub_mul(eta, J, a.b);
  const Vec<S, NX> y = lu_solve(lu, w);
  const Mat<S, NX, NX> yj = lu_solve(lu, J);
  const Mat<S, NX, NX> v = mul(yj, a.A);
  eta = mul_tn_add(a.A, y, a.eta);
  J = mul_tn_sym_add(a.A, v, a.J);
}

template <typename S, int NX, int NY>
__global__ void __launch_bounds__(kStageNT, 2)
    k_bwd_finish(ModelView<S> ms, const __grid_constant__ StageMaps maps, long long T,
                 long long L, long long nchunks, long long nfull, const S* suf, long long suf_cap,
                 ChunkOrder bord, const S* fst, long long fcap, S* mean, S* cov,
                 const S* carry, const S* fmean, const S* fcov, unsigned* err) {
  extern __shared__ __align__(1024) unsigned char fsm[];
  using St = FilterStage<S, NX, NY>;
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = c < nchunks;
  unsigned e = 0;
  const long long k0 = c * L;
  const long long k1 = min(k0 + L, T);
  const long long cta0 = (long long)blockIdx.x * kStageNT;
  const long long jn = min(L, T - cta0 * L);  // CTA-uniform (slots of the CTA's first chunk)
  Vec<S, NX> eta = zeros<S, NX, 1>();
  Mat<S, NX, NX> J = zeros<S, NX, NX>();
  if (live && carry != nullptr) {
    // time-sharded backward pass: (eta, J) of the later shards' backward
    // elements folded (the backward information of everything after this
    // shard); the shard's own suffix of chunk c+1 is applied on top of it
    eta = load_soa<S, NX, 1>(carry, 1);
    J = load_soa<S, NX, NX>(carry + NX, 1);
    if (c + 1 < nchunks) {
      const FElem<S, NX> a = fe_load<S, NX>(suf, suf_cap, bord.at(c + 1));
      bwd_info_apply(a, eta, J, e);
    }
  } else if (live && c + 1 < nchunks) {
    const long long q = bord.at(c + 1);
    eta = load_soa<S, NX, 1>(suf + FLayout<NX>::eta * suf_cap + q, suf_cap);
    J = load_soa<S, NX, NX>(suf + FLayout<NX>::J * suf_cap + q, suf_cap);
  }
  staged_walk_rev<S, NX, NY>(fsm, maps, ms, L, nfull, jn, k0, k1,
                             [&](long long i, bool has, const St& in) {
    if (has) {
      // (eta, J) of a (x) s for the element a of ms step i (Lemma 1, eta / J
      // rows only: they depend on the right operand through (eta, J) alone)
      FElem<S, NX> a = fe_identity<S, NX>();
      const Mat<S, NX, NX> F = in.F();
      a.A = F;
      a.b = in.u();
      a.C = in.Q();
      cond_update(a, in.meas(), e);
      bwd_info_apply(a, eta, J, e);
    }
    // two-filter combination: (I + P J)^-1 (x + P eta), (I + P J)^-1 P
    Vec<S, NX> x;
    Mat<S, NX, NX> P;
    if (fmean != nullptr) {  // dense forward states of another device's forward pass
      x = load<S, NX, 1>(fmean + i * NX);
      P = load<S, NX, NX>(fcov + i * NX * NX);
    } else {
      state_load(fst + (i - k0) * StateLayout<NX>::size * fcap + c, fcap, x, P);
    }
    Mat<S, NX, NX> mm = mul(P, J);
#pragma unroll
    for (int q = 0; q < NX; ++q) mm.a[q][q] += S(1);
    const LU<S, NX> lu = lu_factor(mm, e);
    const Vec<S, NX> rhs = mul_add(P, eta, x);
    const Vec<S, NX> xs = lu_solve(lu, rhs);
    Mat<S, NX, NX> ps = lu_solve(lu, P);
    symmetrize(ps);
    store_state(mean, cov, i, xs, ps);
  });
  if (e) atomicOr(err, e);
}

// one packed element (row-major fields, FLayout / SLayout order) from slot i
// of an SoA buffer
template <typename S>
__global__ void k_extract_elem(const S* buf, long long cap, long long i, int size,
                               S* out) {
  for (int c = threadIdx.x; c < size; c += blockDim.x) out[c] = buf[c * cap + i];
}

// Fold of `count` packed filter elements, left to right (non-commutative);
// the first contains a_1 (A = 0), so the result is a state: out = (b | C).
template <typename S, int NX>
__global__ void k_fold_filter(const S* aggs, int count, S* out, unsigned* err) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  unsigned e = 0;
  constexpr int FS = FLayout<NX>::size;
  FElem<S, NX> acc = fe_load<S, NX>(aggs, 1, 0);
  for (int k = 1; k < count; ++k) acc = filter_combine(acc, fe_load<S, NX>(aggs + k * FS, 1, 0), e);
  for (int i = 0; i < NX; ++i) out[i] = acc.b.a[i][0];
  for (int i = 0; i < NX; ++i)
    for (int j = 0; j < NX; ++j) out[NX + i * NX + j] = acc.C.a[i][j];
  if (e) atomicOr(err, e);
}
// Fold of `count` packed backward (shifted filter) elements, left to right:
// the backward information (eta | J) of the later shards of a sharded PTFS.
template <typename S, int NX>
__global__ void k_fold_backward(const S* aggs, int count, S* out, unsigned* err) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  unsigned e = 0;
  constexpr int FS = FLayout<NX>::size;
  FElem<S, NX> acc = fe_load<S, NX>(aggs, 1, 0);
  for (int k = 1; k < count; ++k) acc = filter_combine(acc, fe_load<S, NX>(aggs + k * FS, 1, 0), e);
  for (int i = 0; i < NX; ++i) out[i] = acc.eta.a[i][0];
  for (int i = 0; i < NX; ++i)
    for (int j = 0; j < NX; ++j) out[NX + i * NX + j] = acc.J.a[i][j];
  if (e) atomicOr(err, e);
}
// Fold of `count` packed smoother elements, left to right; the last contains
// a_T (E = 0), so the result is a state: out = (g | L).
template <typename S, int NX>
__global__ void k_fold_smoother(const S* aggs, int count, S* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  constexpr int SS = SLayout<NX>::size;
  SElem<S, NX> acc = se_load<S, NX>(aggs + (count - 1) * SS, 1, 0);
  for (int k = count - 2; k >= 0; --k) acc = smoother_combine(se_load<S, NX>(aggs + k * SS, 1, 0), acc);
  for (int i = 0; i < NX; ++i) out[i] = acc.g.a[i][0];
  for (int i = 0; i < NX; ++i)
    for (int j = 0; j < NX; ++j) out[NX + i * NX + j] = acc.L.a[i][j];
}

// padding slots [from, to) <- identity
template <class Ops>
__global__ void k_fill_identity(Ops ops, ElemBuf<typename Ops::S> b,
                                long long from, long long to) {
  const long long i = from + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < to) ops.identity(b, i);
}

}  // namespace psk
