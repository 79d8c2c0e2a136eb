// psk_exact.cu -- exact mode: the reference's level-by-level algorithm on the
// GPU with the reference's floating-point operation order.
//
// This translation unit is compiled with --fmad=false (no FMA contraction);
// IEEE +,-,*,/ and sqrt are correctly rounded on both sides, pivots are chosen
// by the same comparisons and there is no reassociation, so results are
// bitwise equal to the reference compiled with -ffp-contract=off (checked by
// tests/test_gpu_parity.py against oracle/_ref).  Dimensions are runtime
// (1..16, mat.hpp:19); matrices live in per-thread local arrays sized by the
// template bound D (4 or 16).
#include <cuda_runtime.h>

#include "psk_common.cuh"
#include "psk_exact.h"
#include "psk_levels.cuh"
#include "psk_mat.cuh"

namespace psk {
namespace ex {

// ---- mat.hpp restatement (runtime dims, reference operation order) -------
template <typename S>
__device__ void mzero(S* a, int n) {
  for (int i = 0; i < n; ++i) a[i] = S(0);
}
template <typename S>
__device__ void mcopy(S* o, const S* a, int n) {
  for (int i = 0; i < n; ++i) o[i] = a[i];
}
template <typename S>
__device__ void madd(S* o, const S* a, const S* b, int n) {  // mat.hpp:84-91
  for (int i = 0; i < n; ++i) o[i] = a[i] + b[i];
}
template <typename S>
__device__ void msub(S* o, const S* a, const S* b, int n) {  // mat.hpp:93-99
  for (int i = 0; i < n; ++i) o[i] = a[i] - b[i];
}
// mat.hpp:101-114
template <typename S>
__device__ void mmul(S* o, const S* a, const S* b, int ar, int ac, int bc) {
  for (int i = 0; i < ar; ++i)
    for (int j = 0; j < bc; ++j) {
      S acc = a[i * ac] * b[j];
      for (int k = 1; k < ac; ++k) acc += a[i * ac + k] * b[k * bc + j];
      o[i * bc + j] = acc;
    }
}
// a^T b (kalman_seq.hpp mat_mul_tn: same products as a materialised
// transpose followed by mat_mul)
template <typename S>
__device__ void mmul_tn(S* o, const S* a, int ar, int ac, const S* b, int bc) {
  for (int i = 0; i < ac; ++i)
    for (int j = 0; j < bc; ++j) {
      S acc = a[i] * b[j];
      for (int k = 1; k < ar; ++k) acc += a[k * ac + i] * b[k * bc + j];
      o[i * bc + j] = acc;
    }
}
// a b^T (kalman_seq.hpp mat_mul_nt)
template <typename S>
__device__ void mmul_nt(S* o, const S* a, int ar, int ac, const S* b, int br) {
  for (int i = 0; i < ar; ++i)
    for (int j = 0; j < br; ++j) {
      S acc = a[i * ac] * b[j * ac];
      for (int k = 1; k < ac; ++k) acc += a[i * ac + k] * b[j * ac + k];
      o[i * br + j] = acc;
    }
}
template <typename S>
__device__ void mtrans(S* o, const S* a, int r, int c) {  // mat.hpp:116-122
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) o[j * r + i] = a[i * c + j];
}
template <typename S>
__device__ void msym(S* a, int n) {  // mat.hpp:124-136
  const S half = S(0.5);
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      S m = (a[i * n + j] + a[j * n + i]) * half;
      a[i * n + j] = m;
      a[j * n + i] = m;
    }
}
template <typename S>
__device__ bool chol(S* out, const S* a, int n) {  // mat.hpp:153-175
  mzero(out, n * n);
  for (int j = 0; j < n; ++j) {
    S diag = a[j * n + j];
    for (int k = 0; k < j; ++k) diag -= out[j * n + k] * out[j * n + k];
    if (!((double)diag > 0.0)) return false;
    S ljj = ssqrt(diag);
    out[j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      S acc = a[i * n + j];
      for (int k = 0; k < j; ++k) acc -= out[i * n + k] * out[j * n + k];
      out[i * n + j] = acc / ljj;
    }
  }
  return true;
}
template <typename S>
__device__ bool lu_factor(S* a, int n, int* perm) {  // mat.hpp:177-205
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    double best = fabs((double)a[c * n + c]);
    for (int r = c + 1; r < n; ++r) {
      double x = fabs((double)a[r * n + c]);
      if (x > best) {
        best = x;
        piv = r;
      }
    }
    if (best == 0.0) return false;
    if (piv != c) {
      for (int j = 0; j < n; ++j) {
        S t = a[c * n + j];
        a[c * n + j] = a[piv * n + j];
        a[piv * n + j] = t;
      }
      int t = perm[c];
      perm[c] = perm[piv];
      perm[piv] = t;
    }
    for (int r = c + 1; r < n; ++r) {
      S f = a[r * n + c] / a[c * n + c];
      a[r * n + c] = f;
      for (int j = c + 1; j < n; ++j) a[r * n + j] -= f * a[c * n + j];
    }
  }
  return true;
}
template <typename S, int D>
__device__ void lu_solve(const S* lu, const int* perm, int n, const S* b,
                         int bc, S* out) {  // mat.hpp:207-228
  for (int col = 0; col < bc; ++col) {
    S y[D];
    for (int i = 0; i < n; ++i) y[i] = b[perm[i] * bc + col];
    for (int i = 1; i < n; ++i)
      for (int k = 0; k < i; ++k) y[i] -= lu[i * n + k] * y[k];
    for (int i = n - 1; i >= 0; --i) {
      for (int k = i + 1; k < n; ++k) y[i] -= lu[i * n + k] * y[k];
      y[i] /= lu[i * n + i];
    }
    for (int i = 0; i < n; ++i) out[i * bc + col] = y[i];
  }
}
template <typename S, int D>
__device__ bool solve_spd(const S* a, int n, const S* b, int bc,
                          S* out) {  // mat.hpp:244-269
  S l[D * D];
  if (!chol(l, a, n)) return false;
  for (int col = 0; col < bc; ++col) {
    S y[D];
    for (int i = 0; i < n; ++i) {
      S acc = b[i * bc + col];
      for (int k = 0; k < i; ++k) acc -= l[i * n + k] * y[k];
      y[i] = acc / l[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      S acc = y[i];
      for (int k = i + 1; k < n; ++k) acc -= l[k * n + i] * y[k];
      y[i] = acc / l[i * n + i];
    }
    for (int i = 0; i < n; ++i) out[i * bc + col] = y[i];
  }
  return true;
}

// ---- element storage (SoA, runtime nx) ------------------------------------
// filter element components: A | b | C | eta | J  (FLayout packing)
struct FOff {
  int A, b, C, eta, J, size;
  __device__ explicit FOff(int nx)
      : A(0), b(nx * nx), C(nx * nx + nx), eta(2 * nx * nx + nx),
        J(2 * nx * nx + 2 * nx), size(3 * nx * nx + 2 * nx) {}
};
struct SOff {
  int E, g, L, size;
  __device__ explicit SOff(int nx)
      : E(0), g(nx * nx), L(nx * nx + nx), size(2 * nx * nx + nx) {}
};
template <typename S>
__device__ void gather(S* o, const ElemBuf<S>& b, long long i, int off, int n) {
  for (int c = 0; c < n; ++c) o[c] = b.p[(long long)(off + c) * b.cap + i];
}
template <typename S>
__device__ void scatter(const ElemBuf<S>& b, long long i, int off, const S* v,
                        int n) {
  for (int c = 0; c < n; ++c) b.p[(long long)(off + c) * b.cap + i] = v[c];
}

template <typename S>
struct MV {  // model accessors with strides (lgssm.hpp:5-8)
  const ModelView<S>& m;
  __device__ const S* f(long long k) const { return m.f + k * m.sf; }
  __device__ const S* u(long long k) const { return m.u + k * m.su; }
  __device__ const S* q(long long k) const { return m.q + k * m.sq; }
  __device__ const S* h(long long k) const { return m.h + k * m.sh; }
  __device__ const S* d(long long k) const { return m.d + k * m.sd; }
  __device__ const S* r(long long k) const { return m.r + k * m.sr; }
  __device__ const S* y(long long k) const { return m.y + k * m.sy; }
};

// kalman_seq.hpp:36-56 with (F,u,Q)[k-1]
template <typename S, int D>
__device__ void kf_predict(const ModelView<S>& m, long long k, const S* x,
                           const S* p, S* ox, S* op) {
  MV<S> a{m};
  const int nx = m.nx;
  const S* f = a.f(k - 1);
  mmul(ox, f, x, nx, nx, 1);
  madd(ox, ox, a.u(k - 1), nx);
  S fp[D * D];
  mmul(fp, f, p, nx, nx, nx);
  mmul_nt(op, fp, nx, nx, f, nx);
  madd(op, op, a.q(k - 1), nx * nx);
  msym(op, nx);
}

// kalman_elems.hpp:51-149 (k 1-based); writes packed element into e
template <typename S, int D>
__device__ __noinline__ unsigned make_filter_element(const ModelView<S>& m, long long k,
                                        S* ea, S* eb, S* ec, S* eeta, S* ej) {
  MV<S> acc{m};
  const int nx = m.nx, ny = m.ny;
  const S* h = acc.h(k - 1);
  const S* d = acc.d(k - 1);
  const S* r = acc.r(k - 1);
  const S* f = acc.f(k - 1);
  const S* y = acc.y(k - 1);
  S sk[D * D], v[D], s1[D * D], s2[D * D], s3[D * D], s4[D * D], s5[D * D];
  if (k == 1) {
    S pxm[D], pxp[D * D];
    kf_predict<S, D>(m, 1, m.m0, m.p0, pxm, pxp);
    mmul(s1, h, pxp, ny, nx, nx);
    mmul_nt(sk, s1, ny, nx, h, ny);
    madd(sk, sk, r, ny * ny);
    msym(sk, ny);
    if (!solve_spd<S, D>(sk, ny, s1, nx, s2)) return kErrNotPD;
    mtrans(s3, s2, ny, nx);
    mmul(v, h, pxm, ny, nx, 1);
    msub(v, y, v, ny);
    msub(v, v, d, ny);
    mzero(ea, nx * nx);
    mmul(eb, s3, v, nx, ny, 1);
    madd(eb, eb, pxm, nx);
    mmul(s4, s3, sk, nx, ny, ny);
    mmul_nt(s5, s4, nx, ny, s3, nx);
    msub(ec, pxp, s5, nx * nx);
    msym(ec, nx);
  } else {
    const S* q = acc.q(k - 1);
    const S* u = acc.u(k - 1);
    mmul(s1, h, q, ny, nx, nx);
    mmul_nt(sk, s1, ny, nx, h, ny);
    madd(sk, sk, r, ny * ny);
    msym(sk, ny);
    if (!solve_spd<S, D>(sk, ny, s1, nx, s2)) return kErrNotPD;
    mtrans(s3, s2, ny, nx);
    mmul(s4, s3, h, nx, ny, nx);
    mmul(s5, s4, f, nx, nx, nx);
    msub(ea, f, s5, nx * nx);
    mmul(v, h, u, ny, nx, 1);
    msub(v, y, v, ny);
    msub(v, v, d, ny);
    mmul(eb, s3, v, nx, ny, 1);
    madd(eb, eb, u, nx);
    mmul(s5, s4, q, nx, nx, nx);
    msub(ec, q, s5, nx * nx);
    msym(ec, nx);
  }
  if (!solve_spd<S, D>(sk, ny, v, 1, s1)) return kErrNotPD;
  mmul_tn(s2, h, ny, nx, s1, 1);
  mmul_tn(eeta, f, nx, nx, s2, 1);
  mmul(s2, h, f, ny, nx, nx);
  if (!solve_spd<S, D>(sk, ny, s2, nx, s3)) return kErrNotPD;
  mmul_tn(s4, s2, ny, nx, s3, nx);
  mcopy(ej, s4, nx * nx);
  msym(ej, nx);
  return 0;
}

// kalman_elems.hpp:151-193 (k 1-based)
template <typename S, int D>
__device__ __noinline__ unsigned make_smoother_element(const ModelView<S>& m,
                                          const S* x, const S* p, long long k,
                                          S* ee, S* eg, S* el) {
  MV<S> acc{m};
  const int nx = m.nx;
  if (k == m.t) {
    mzero(ee, nx * nx);
    mcopy(eg, x, nx);
    mcopy(el, p, nx * nx);
    return 0;
  }
  const S* f = acc.f(k);
  const S* q = acc.q(k);
  const S* u = acc.u(k);
  S fp[D * D], pp[D * D], et[D * D], fx[D], efp[D * D];
  mmul(fp, f, p, nx, nx, nx);
  mmul_nt(pp, fp, nx, nx, f, nx);
  madd(pp, pp, q, nx * nx);
  msym(pp, nx);
  if (!solve_spd<S, D>(pp, nx, fp, nx, et)) return kErrNotPD;
  mtrans(ee, et, nx, nx);
  mmul(fx, f, x, nx, nx, 1);
  madd(fx, fx, u, nx);
  mmul(eg, ee, fx, nx, nx, 1);
  msub(eg, x, eg, nx);
  mmul(fp, f, p, nx, nx, nx);
  mmul(efp, ee, fp, nx, nx, nx);
  msub(el, p, efp, nx * nx);
  msym(el, nx);
  return 0;
}

// ---- operator policies for k_level ---------------------------------------
template <typename S_, int D>
struct ExactFilterOps {
  using S = S_;
  int nx;
  unsigned* err;
  // kalman_elems.hpp:266-336, Lemma 1 (writes at the end: alias-safe)
  __device__ __noinline__ void combine(const ElemBuf<S>& dst, long long di,
                          const ElemBuf<S>& lb, long long li,
                          const ElemBuf<S>& rb, long long ri) const {
    const FOff o(nx);
    const int n2 = nx * nx;
    S la[D * D], lbv[D], lc[D * D], leta[D], lj[D * D];
    S ra[D * D], rbv[D], rc[D * D], reta[D], rj[D * D];
    gather(la, lb, li, o.A, n2);
    gather(lbv, lb, li, o.b, nx);
    gather(lc, lb, li, o.C, n2);
    gather(leta, lb, li, o.eta, nx);
    gather(lj, lb, li, o.J, n2);
    gather(ra, rb, ri, o.A, n2);
    gather(rbv, rb, ri, o.b, nx);
    gather(rc, rb, ri, o.C, n2);
    gather(reta, rb, ri, o.eta, nx);
    gather(rj, rb, ri, o.J, n2);
    S mm[D * D], nn[D * D], x1[D * D], na[D * D], bc[D], x2[D], nb[D];
    int mperm[D], nperm[D];
    mmul(mm, lc, rj, nx, nx, nx);
    for (int i = 0; i < nx; ++i) mm[i * nx + i] += S(1);
    if (!lu_factor(mm, nx, mperm)) {
      atomicOr(err, kErrSingular);
      return;
    }
    mmul(nn, rj, lc, nx, nx, nx);
    for (int i = 0; i < nx; ++i) nn[i * nx + i] += S(1);
    if (!lu_factor(nn, nx, nperm)) {
      atomicOr(err, kErrSingular);
      return;
    }
    lu_solve<S, D>(mm, mperm, nx, la, nx, x1);
    mmul(na, ra, x1, nx, nx, nx);
    mmul(bc, lc, reta, nx, nx, 1);
    madd(bc, bc, lbv, nx);
    lu_solve<S, D>(mm, mperm, nx, bc, 1, x2);
    mmul(nb, ra, x2, nx, nx, 1);
    madd(nb, nb, rbv, nx);
    // C'
    S nc[D * D];
    lu_solve<S, D>(mm, mperm, nx, lc, nx, x1);  // x3
    {
      S ac[D * D];
      mmul(ac, ra, x1, nx, nx, nx);
      mmul_nt(nc, ac, nx, nx, ra, nx);
    }
    madd(nc, nc, rc, n2);
    msym(nc, nx);
    // eta'
    S ne[D];
    {
      S jb[D], y1[D];
      mmul(jb, rj, lbv, nx, nx, 1);
      msub(jb, reta, jb, nx);
      lu_solve<S, D>(nn, nperm, nx, jb, 1, y1);
      mmul_tn(ne, la, nx, nx, y1, 1);
      madd(ne, ne, leta, nx);
    }
    // J'
    S nj[D * D];
    {
      lu_solve<S, D>(nn, nperm, nx, rj, nx, x1);  // y2
      S ja[D * D];
      mmul(ja, x1, la, nx, nx, nx);
      mmul_tn(nj, la, nx, nx, ja, nx);
      madd(nj, nj, lj, n2);
      msym(nj, nx);
    }
    scatter(dst, di, o.A, na, n2);
    scatter(dst, di, o.b, nb, nx);
    scatter(dst, di, o.C, nc, n2);
    scatter(dst, di, o.eta, ne, nx);
    scatter(dst, di, o.J, nj, n2);
  }
  __device__ void assign(const ElemBuf<S>& d, long long di,
                         const ElemBuf<S>& s, long long si) const {
    const int n = FOff(nx).size;
    for (int c = 0; c < n; ++c) d.p[(long long)c * d.cap + di] = s.p[(long long)c * s.cap + si];
  }
  __device__ void identity(const ElemBuf<S>& d, long long di) const {
    const FOff o(nx);
    for (int c = 0; c < o.size; ++c) d.p[(long long)c * d.cap + di] = S(0);
    for (int i = 0; i < nx; ++i) d.p[(long long)(o.A + i * nx + i) * d.cap + di] = S(1);
  }
};

template <typename S_, int D>
struct ExactSmootherOps {
  using S = S_;
  int nx;
  unsigned* err;
  // kalman_elems.hpp:395-418, Lemma 2
  __device__ __noinline__ void combine(const ElemBuf<S>& dst, long long di,
                          const ElemBuf<S>& lb, long long li,
                          const ElemBuf<S>& rb, long long ri) const {
    const SOff o(nx);
    const int n2 = nx * nx;
    S le[D * D], lg[D], ll[D * D], re[D * D], rg[D], rl[D * D];
    gather(le, lb, li, o.E, n2);
    gather(lg, lb, li, o.g, nx);
    gather(ll, lb, li, o.L, n2);
    gather(re, rb, ri, o.E, n2);
    gather(rg, rb, ri, o.g, nx);
    gather(rl, rb, ri, o.L, n2);
    S nei[D * D], ng[D], el[D * D], nl[D * D];
    mmul(nei, le, re, nx, nx, nx);
    mmul(ng, le, rg, nx, nx, 1);
    madd(ng, ng, lg, nx);
    mmul(el, le, rl, nx, nx, nx);
    mmul_nt(nl, el, nx, nx, le, nx);
    madd(nl, nl, ll, n2);
    msym(nl, nx);
    scatter(dst, di, o.E, nei, n2);
    scatter(dst, di, o.g, ng, nx);
    scatter(dst, di, o.L, nl, n2);
  }
  __device__ void assign(const ElemBuf<S>& d, long long di,
                         const ElemBuf<S>& s, long long si) const {
    const int n = SOff(nx).size;
    for (int c = 0; c < n; ++c) d.p[(long long)c * d.cap + di] = s.p[(long long)c * s.cap + si];
  }
  __device__ void identity(const ElemBuf<S>& d, long long di) const {
    const SOff o(nx);
    for (int c = 0; c < o.size; ++c) d.p[(long long)c * d.cap + di] = S(0);
    for (int i = 0; i < nx; ++i) d.p[(long long)(o.E + i * nx + i) * d.cap + di] = S(1);
  }
};

// ---- build / extract kernels (kalman_par.hpp) ------------------------------
// build_filter_elems (shift 0, :29-61) / build_shifted_filter_elems (shift 1,
// :63-89): slot i holds a_{i+1+shift} or the identity
template <typename S, int D>
__global__ void k_build_filter(ModelView<S> m, ElemBuf<S> b, int shift,
                               unsigned* err) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n) return;
  const int nx = m.nx, n2 = nx * nx;
  const FOff o(nx);
  if (i + 1 + shift <= m.t) {
    S ea[D * D], eb[D], ec[D * D], eeta[D], ej[D * D];
    unsigned e = make_filter_element<S, D>(m, i + 1 + shift, ea, eb, ec, eeta, ej);
    if (e) atomicOr(err, e);
    scatter(b, i, o.A, ea, n2);
    scatter(b, i, o.b, eb, nx);
    scatter(b, i, o.C, ec, n2);
    scatter(b, i, o.eta, eeta, nx);
    scatter(b, i, o.J, ej, n2);
  } else {
    ExactFilterOps<S, D>{nx, err}.identity(b, i);
  }
}
// build_smoother_elems (kalman_par.hpp:121-153)
template <typename S, int D>
__global__ void k_build_smoother(ModelView<S> m, const S* fmean,
                                 const S* fcov, ElemBuf<S> b, unsigned* err) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n) return;
  const int nx = m.nx, n2 = nx * nx;
  const SOff o(nx);
  if (i < m.t) {
    S ee[D * D], eg[D], el[D * D];
    unsigned e = make_smoother_element<S, D>(m, fmean + i * nx, fcov + i * n2,
                                             i + 1, ee, eg, el);
    if (e) atomicOr(err, e);
    scatter(b, i, o.E, ee, n2);
    scatter(b, i, o.g, eg, nx);
    scatter(b, i, o.L, el, n2);
  } else {
    ExactSmootherOps<S, D>{nx, err}.identity(b, i);
  }
}
// extraction launches (kalman_par.hpp:91-108, 165-178): comps [o1, o1+nx)
// -> mean, [o2, o2+n2) -> cov
template <typename S>
__global__ void k_extract(ElemBuf<S> b, long long t, int nx, int o1, int o2,
                          S* mean, S* cov) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= t) return;
  for (int c = 0; c < nx; ++c) mean[i * nx + c] = b.p[(long long)(o1 + c) * b.cap + i];
  for (int c = 0; c < nx * nx; ++c)
    cov[i * nx * nx + c] = b.p[(long long)(o2 + c) * b.cap + i];
}
// combine_tf_stats (kalman_par.hpp:181-201) -> tf_combine
// (kalman_seq.hpp:236-260); mean/cov hold the filtered stats on entry
template <typename S, int D>
__global__ void k_tf_combine(ElemBuf<S> bwd, long long t, int nx, S* mean,
                             S* cov, unsigned* err) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= t) return;
  const FOff o(nx);
  const int n2 = nx * nx;
  S x[D], p[D * D], eta[D], jm[D * D], mm[D * D], rhs[D], ox[D], tmp[D * D];
  int perm[D];
  mcopy(x, mean + i * nx, nx);
  mcopy(p, cov + i * n2, n2);
  gather(eta, bwd, i, o.eta, nx);
  gather(jm, bwd, i, o.J, n2);
  mmul(mm, p, jm, nx, nx, nx);
  for (int q = 0; q < nx; ++q) mm[q * nx + q] += S(1);
  if (!lu_factor(mm, nx, perm)) {
    atomicOr(err, kErrSingular);
    return;
  }
  mmul(rhs, p, eta, nx, nx, 1);
  madd(rhs, rhs, x, nx);
  lu_solve<S, D>(mm, perm, nx, rhs, 1, ox);
  lu_solve<S, D>(mm, perm, nx, p, nx, tmp);
  msym(tmp, nx);
  mcopy(mean + i * nx, ox, nx);
  mcopy(cov + i * n2, tmp, n2);
}

}  // namespace ex

// ---- host side -------------------------------------------------------------
namespace {
inline int grid_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148LL * 64) g = 148LL * 64;
  return (int)g;
}
}  // namespace

template <typename S, int D>
static void exact_filter_kernels(ExactLaunch& L, const ModelView<S>& m,
                                 ElemBuf<S> b, int shift) {
  ex::k_build_filter<S, D><<<grid_for(b.n, 128), 128, 0, L.stream>>>(m, b, shift, L.err);
  L.count(shift ? "exact_build_shifted" : "exact_build_filter");
}

template <typename S, int D, template <typename, int> class Ops>
static void exact_scan(ExactLaunch& L, int nx, const ScanPlan& plan,
                       Bufs3<Ops<S, D>> bufs) {
  Ops<S, D> ops{nx, L.err};
  for (const LevelDesc& d : plan.levels) {
    const int g = d.kind == kLvSeqChain ? 1 : grid_for(d.count, 128);
    k_level<Ops<S, D>><<<g, 128, 0, L.stream>>>(ops, bufs, d);
    L.count("exact_scan_level");
  }
}

template <typename S, int D>
static void exact_run_t(ExactLaunch& L, const ModelView<S>& m, int method,
                        const ScanPlan& plan, S* el0, S* el1, S* el2,
                        S* bel0, S* mean, S* cov) {
  const int nx = m.nx;
  const long long n = plan.n;
  const ex::FOff fo(nx);
  const ex::SOff so(nx);
  // ---- forward filter: build -> scan_forward -> extract (kalman_par.hpp:111-119)
  Bufs3<ex::ExactFilterOps<S, D>> fb;
  fb.b[0] = ElemBuf<S>{el0, n, n, 0};
  fb.b[1] = ElemBuf<S>{el1, plan.cap1 ? plan.cap1 : 1, plan.cap1, 0};
  fb.b[2] = ElemBuf<S>{el2, plan.cap2 ? plan.cap2 : 1, plan.cap2, 0};
  exact_filter_kernels<S, D>(L, m, fb.b[0], 0);
  exact_scan<S, D, ex::ExactFilterOps>(L, nx, plan, fb);
  ex::k_extract<S><<<grid_for(m.t, 128), 128, 0, L.stream>>>(fb.b[0], m.t, nx, fo.b, fo.C, mean, cov);
  L.count("exact_extract_filter");
  if (method == 1) {  // PRTS: smoother elements -> scan_reverse -> extract
    Bufs3<ex::ExactSmootherOps<S, D>> sb;
    sb.b[0] = ElemBuf<S>{el0, n, n, 1};
    sb.b[1] = ElemBuf<S>{el1, plan.cap1 ? plan.cap1 : 1, plan.cap1, 1};
    sb.b[2] = ElemBuf<S>{el2, plan.cap2 ? plan.cap2 : 1, plan.cap2, 1};
    ex::k_build_smoother<S, D><<<grid_for(n, 128), 128, 0, L.stream>>>(m, mean, cov, sb.b[0], L.err);
    L.count("exact_build_smoother");
    exact_scan<S, D, ex::ExactSmootherOps>(L, nx, plan, sb);
    ex::k_extract<S><<<grid_for(m.t, 128), 128, 0, L.stream>>>(sb.b[0], m.t, nx, so.g, so.L, mean, cov);
    L.count("exact_extract_smoother");
  } else if (method == 2) {  // PTFS: shifted elements -> scan_reverse -> tf
    Bufs3<ex::ExactFilterOps<S, D>> bb;
    bb.b[0] = ElemBuf<S>{bel0, n, n, 1};
    bb.b[1] = ElemBuf<S>{el1, plan.cap1 ? plan.cap1 : 1, plan.cap1, 1};
    bb.b[2] = ElemBuf<S>{el2, plan.cap2 ? plan.cap2 : 1, plan.cap2, 1};
    exact_filter_kernels<S, D>(L, m, bb.b[0], 1);
    exact_scan<S, D, ex::ExactFilterOps>(L, nx, plan, bb);
    ex::k_tf_combine<S, D><<<grid_for(m.t, 128), 128, 0, L.stream>>>(bb.b[0], m.t, nx, mean, cov, L.err);
    L.count("exact_tf_combine");
  }
}

template <typename S>
void exact_run(ExactLaunch& L, const ModelView<S>& m, int method,
               const ScanPlan& plan, S* el0, S* el1, S* el2, S* bel0, S* mean,
               S* cov) {
  if (m.nx <= 4 && m.ny <= 4)
    exact_run_t<S, 4>(L, m, method, plan, el0, el1, el2, bel0, mean, cov);
  else
    exact_run_t<S, 16>(L, m, method, plan, el0, el1, el2, bel0, mean, cov);
}

template void exact_run<float>(ExactLaunch&, const ModelView<float>&, int,
                               const ScanPlan&, float*, float*, float*, float*,
                               float*, float*);
template void exact_run<double>(ExactLaunch&, const ModelView<double>&, int,
                                const ScanPlan&, double*, double*, double*,
                                double*, double*, double*);

}  // namespace psk
