// psk_tile_impl.cuh -- the register-tiled warp kernels (psk_tile.cuh) for
// compile-time (NX, NY), and their host dispatch.  Launch sequence and
// buffer formats are those of the runtime-dimension wide path
// (psk_wide_impl.cuh), whose warp-per-combine chunk scans are reused:
//   k_t_reduce (conditional Kalman per chunk)  ->  chunk scan (Lemma 1)  ->
//   k_t_finish (filtered stats, or per-step smoothing elements + smoother
//   chunk fold)  ->  reverse chunk scan (Lemma 2)  ->  k_t_smoother_finish.
// Chunk elements are AoS in the reference's field order (FOffs / SOffs); the
// per-step smoothing elements of a PRTS (`egl`, private to the finish and the
// smoother finish) hold E^T in place of E so both kernels read them as
// contiguous rows.
#pragma once
#include <cuda_runtime.h>

#include "psk_tile.cuh"
#include "psk_wide_impl.cuh"

namespace psk {
namespace tile {
using wide::FOffs;
using wide::SOffs;

// Lane tile of an M x N product over the kGW lanes of a chunk: the largest of
// 4x8, 4x4, 2x4, 1x4, 2x2, 1x2, 1x1 that still gives every lane a tile (the
// finest tiling when there are fewer than kGW outputs).
constexpr bool tile_fits(int M, int N, int tm, int tn) {
  return M % tm == 0 && N % tn == 0 && (M / tm) * (N / tn) >= kGW;
}
constexpr int pick_tm(int M, int N) {
  return tile_fits(M, N, 4, 8) ? 4 : tile_fits(M, N, 4, 4) ? 4 : tile_fits(M, N, 2, 4) ? 2
       : tile_fits(M, N, 1, 4) ? 1 : tile_fits(M, N, 2, 2) ? 2 : 1;
}
constexpr int pick_tn(int M, int N) {
  return tile_fits(M, N, 4, 8) ? 8 : tile_fits(M, N, 4, 4) ? 4 : tile_fits(M, N, 2, 4) ? 4
       : tile_fits(M, N, 1, 4) ? 4 : tile_fits(M, N, 2, 2) ? 2 : tile_fits(M, N, 1, 2) ? 2 : 1;
}
template <int M, int N>
struct Pick {
  static constexpr int TM = pick_tm(M, N), TN = pick_tn(M, N);
  static_assert((M / TM) * (N / TN) <= kGW, "one tile per lane");
};

// ---- per-warp frames (scalars; every offset a whole number of 16 bytes) -------
// Bank placement: the fused products read rows of two matrices side by side
// ([A | C] and [HC | HA]); their bases sit 16 bytes apart modulo 128 so the
// two halves of a 16-byte load phase never share a bank.
template <typename S, int N, int M>
struct RFrame {  // reduce
  static constexpr int V = vec16<S>();  // 16 bytes in scalars
  static constexpr int LD = ldpad<S>(N), MAT = N * LD;
  static constexpr int HAO = N + V;  // column of HA inside an HCA row
  static constexpr int LDH = ldpad<S>(HAO + N), LDA = ldpad<S>(M + 2 * N + 1);
  // T (F C, column-major) is live from the prediction to C's update only, the
  // measurement blocks HCA / AUG after it: they share one region
  static constexpr int A0 = 0, A1 = MAT, C = 2 * MAT + V, J = 3 * MAT + 2 * V,
                       T = 4 * MAT + 2 * V, HCA = T, AUG = HCA + M * LDH,
                       REnd = (AUG + M * LDA > T + MAT) ? AUG + M * LDA : T + MAT,
                       b = REnd, eta = b + up16<S>(N),
                       tmp = eta + up16<S>(N), vv = tmp + up16<S>(N), pv = vv + up16<S>(M),
                       size = pv + 2 * up16<S>(N > M ? N : M);
};
template <typename S, int N, int M>
struct FFrame {  // finish
  static constexpr int LD = ldpad<S>(N), MAT = N * LD;
  static constexpr int LD2 = ldpad<S>(2 * N), LDP = ldpad<S>(N), LDA3 = ldpad<S>(M + N + 1);
  // FP (column-major; later the fold's T = E_a L) is dead before the update's
  // HP / [S | HP | v] blocks are formed: they share one region.  Three slots
  // rotate between the filtered P, the predicted PP and the chunk's E_a.
  static constexpr int P0 = 0, P1 = MAT, Ea0 = 2 * MAT, FPt = 3 * MAT, HP = FPt,
                       AUG3 = HP + M * LDP,
                       REnd = (AUG3 + M * LDA3 > FPt + MAT) ? AUG3 + M * LDA3 : FPt + MAT,
                       La = REnd, AUG2 = La + MAT,
                       x = AUG2 + N * LD2, xp = x + up16<S>(N), g = xp + up16<S>(N),
                       ga = g + up16<S>(N), vv = ga + up16<S>(N), pv = vv + up16<S>(M),
                       size = pv + 2 * up16<S>(N > M ? N : M);
};
template <typename S, int N>
struct SFrame {  // smoother finish
  static constexpr int LD = ldpad<S>(N), MAT = N * LD;
  static constexpr int Ps = 0, Tt = MAT, Et = 2 * MAT, Lk = 3 * MAT, xs = 4 * MAT,
                       tmp = xs + up16<S>(N), g = tmp + up16<S>(N), size = g + up16<S>(N);
};

// chunks (lane groups) per CTA of each kernel: two CTAs per SM fit in shared
// memory (reduce 12, finish 8, smoother finish 16 chunks per SM)
constexpr int kGroupsReduce = 7, kGroupsFinish = 6, kGroupsSmooth = 8;

template <typename S, int N, int M, int FR, int G>
__host__ __device__ constexpr int cta_smem(bool invariant) {
  return (int)sizeof(S) *
         (G * (FR + (invariant ? 0 : ModelFrame<S, N, M>::size)) +
          (invariant ? ModelFrame<S, N, M>::size : 0));
}

// this warp's frame and its model frame; the CTA-wide model of a
// time-invariant series is loaded here (one barrier)
template <typename S, int N, int M, int FR>
__device__ __forceinline__ void frames(const ModelView<S>& m, bool inv, S*& fr, S*& mf) {
  extern __shared__ __align__(16) unsigned char tsm[];
  S* base = reinterpret_cast<S*>(tsm);
  const int w = threadIdx.x / kGW;
  constexpr int MS = ModelFrame<S, N, M>::size;
  if (inv) {
    mf = base;
    fr = base + MS + w * FR;
    if (w == 0) load_model<S, N, M>(mf, m, 0);
    __syncthreads();
  } else {
    fr = base + w * (FR + MS);
    mf = fr + FR;
  }
}

// ---- reduce: chunk c -> one filtering element (A, b, C, eta, J) --------------
// The conditional-Kalman recursion of psk_fast.cuh (k_filter_reduce) with
// warp-tiled products; from the identity (or the prior in state form for the
// chunk holding step 1, kalman_elems.hpp:68-96).
template <typename S, int N, int M>
__global__ void __launch_bounds__(kGW * kGroupsReduce)
    k_t_reduce(ModelView<S> m, long long L, long long nchunks, S* agg, unsigned* err) {
  using RF = RFrame<S, N, M>;
  using MF = ModelFrame<S, N, M>;
  constexpr int LD = RF::LD, LDH = RF::LDH, LDA = RF::LDA, LDM = MF::LDM, LDR = MF::LDR;
  const bool inv = time_invariant(m);
  S *fr, *mf;
  frames<S, N, M, RF::size>(m, inv, fr, mf);
  const long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / kGW;
  if (c >= nchunks) return;  // warp-uniform (after the CTA barrier)
  const int ln = lane();
  unsigned e = 0;
  const long long k0 = c * L, k1 = min(k0 + L, m.t);
  const bool prior = k0 == 0 && m.prior_first;
  S* A = fr + RF::A0;
  S* An = fr + RF::A1;
  S* C = fr + RF::C;
  S* T = fr + RF::T;
  S* J = fr + RF::J;
  S* HCA = fr + RF::HCA;
  S* AUG = fr + RF::AUG;
  S* b = fr + RF::b;
  S* eta = fr + RF::eta;
  S* tmp = fr + RF::tmp;
  S* vv = fr + RF::vv;
  S* pv = fr + RF::pv;
  for (int i = ln; i < N * N; i += kGW) {
    const int r = i / N, cc = i % N;
    A[r * LD + cc] = (!prior && r == cc) ? S(1) : S(0);
    C[r * LD + cc] = prior ? m.p0[i] : S(0);
    J[r * LD + cc] = S(0);
  }
  if (ln < N) {
    b[ln] = prior ? m.m0[ln] : S(0);
    eta[ln] = S(0);
  }
  gsync();
  const S* Fc = mf + MF::Fc;
  const S* Qm = mf + MF::Q;
  const S* Ht = mf + MF::Ht;
  const S* Rm = mf + MF::R;
  for (long long k = k0; k < k1; ++k) {
    if (!inv) {
      load_model<S, N, M>(mf, m, k);
      gsync();
    }
    // predict the conditional: [A' | T] = F [A | C] (T = F C, column-major)
    {
      using P = Pick<N, 2 * N>;
      using TL = Tiling<N, 2 * N, P::TM, P::TN>;
      if (TL::active()) {
        const int r0 = TL::r0(), c0 = TL::c0();
        S acc[P::TM][P::TN];
        zero(acc);
        const bool left = c0 < N;
        const S* rp = left ? A + c0 : C + (c0 - N);
        mma<N, P::TM, P::TN, 1, LD, LD, 1>(acc, Fc + r0, rp);
        if (left)
          put<P::TM, P::TN, LD, 1>(An + r0 * LD + c0, acc);
        else
          put<P::TM, P::TN, 1, LD>(T + (c0 - N) * LD + r0, acc);
      }
      if (ln < N) tmp[ln] = mf[MF::u + ln] + matvec_row<N, N, 1, LD>(Fc, b, ln);
    }
    gsync();
    {  // C = (F C) F^T + Q
      using P = Pick<N, N>;
      using TL = Tiling<N, N, P::TM, P::TN>;
      if (TL::active()) {
        const int r0 = TL::r0(), c0 = TL::c0();
        S acc[P::TM][P::TN];
        init<P::TM, P::TN, LD, 1>(acc, Qm + r0 * LD + c0);
        mma<N, P::TM, P::TN, 1, LD, LD, 1>(acc, T + r0, Fc + c0);
        put<P::TM, P::TN, LD, 1>(C + r0 * LD + c0, acc);  // symmetrised by the update
      }
      if (ln < N) b[ln] = tmp[ln];
    }
    {
      S* t = A;
      A = An;
      An = t;
    }
    gsync();
    // [HC | HA] = H [C | A] -> HCA and the augmented block
    {
      using P = Pick<M, 2 * N>;
      using TL = Tiling<M, 2 * N, P::TM, P::TN>;
      if (TL::active()) {
        const int r0 = TL::r0(), c0 = TL::c0();
        S acc[P::TM][P::TN];
        zero(acc);
        const S* rp = c0 < N ? C + c0 : A + (c0 - N);
        mma<N, P::TM, P::TN, 1, LDM, LD, 1>(acc, Ht + r0, rp);
        put<P::TM, P::TN, LDH, 1>(HCA + r0 * LDH + (c0 < N ? c0 : c0 - N + RF::HAO), acc);
        put<P::TM, P::TN, LDA, 1>(AUG + r0 * LDA + M + c0, acc);
      }
      if (ln < M) {  // v = y - H b - d
        const S y = inv ? m.Y(k)[ln] : mf[MF::y + ln];
        const S v = y - mf[MF::d + ln] - matvec_row<M, N, 1, LDM>(Ht, b, ln);
        vv[ln] = v;
        AUG[ln * LDA + M + 2 * N] = v;
      }
    }
    gsync();
    {  // S = HC H^T + R
      using P = Pick<M, M>;
      using TL = Tiling<M, M, P::TM, P::TN>;
      if (TL::active()) {
        const int r0 = TL::r0(), c0 = TL::c0();
        S acc[P::TM][P::TN];
        init<P::TM, P::TN, LDR, 1>(acc, Rm + r0 * LDR + c0);
        mma<N, P::TM, P::TN, LDH, 1, LDM, 1>(acc, HCA + r0 * LDH, Ht + c0);
        put_sym<P::TM, P::TN, LDA>(AUG, acc, r0, c0);
      }
    }
    gsync();
    gj_spd<M, M + 2 * N + 1, LDA>(AUG, pv, e);  // [I | K^T | S^-1 HA | S^-1 v]
    {  // J += HA^T S^-1 HA
      using P = Pick<N, N>;
      using TL = Tiling<N, N, P::TM, P::TN>;
      if (TL::active()) {
        const int r0 = TL::r0(), c0 = TL::c0();
        S acc[P::TM][P::TN];
        init<P::TM, P::TN, LD, 1>(acc, J + r0 * LD + c0);
        mma<M, P::TM, P::TN, 1, LDH, LDA, 1>(acc, HCA + RF::HAO + r0, AUG + M + N + c0);
        put_sym<P::TM, P::TN, LD>(J, acc, r0, c0);
      }
    }
    {  // [A | C] -= K [HA | HC]
      using P = Pick<N, 2 * N>;
      using TL = Tiling<N, 2 * N, P::TM, P::TN>;
      if (TL::active()) {
        const int r0 = TL::r0(), c0 = TL::c0();
        S acc[P::TM][P::TN];
        const bool left = c0 < N;
        S* dst = left ? A + r0 * LD + c0 : C + r0 * LD + (c0 - N);
        init<P::TM, P::TN, LD, 1>(acc, dst);
        const S* rp = left ? HCA + RF::HAO + c0 : HCA + (c0 - N);
        mma<M, P::TM, P::TN, 1, LDA, LDH, 1, true>(acc, AUG + M + r0, rp);
        if (left)
          put<P::TM, P::TN, LD, 1>(dst, acc);
        else
          put_sym<P::TM, P::TN, LD>(C, acc, r0, c0 - N);
      }
    }
    if (ln < N) {  // b += K v ; eta += HA^T S^-1 v
      S s = b[ln], h = eta[ln];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        s = sfma(AUG[q * LDA + M + ln], vv[q], s);
        h = sfma(HCA[q * LDH + RF::HAO + ln], AUG[q * LDA + M + 2 * N], h);
      }
      b[ln] = s;
      eta[ln] = h;
    }
    gsync();
  }
  const FOffs F(N);
  S* o = agg + c * F.size;
  gstore_mat<N, LD, false, false>(o + F.A, A);
  gstore_mat<N, LD, false, true>(o + F.C, C);
  gstore_mat<N, LD, false, true>(o + F.J, J);
  if (ln < N) {
    o[F.b + ln] = b[ln];
    o[F.eta + ln] = eta[ln];
  }
  if (e && ln == 0) atomicOr(err, e);
}

// ---- finish ------------------------------------------------------------------
// Prediction from the filtered (x, P) in (x, P slot) with step-k blocks in the
// model frame: FP (FPt column-major and the right half of AUG2), PP = FP F^T +
// Q (left half of AUG2 and the Pn slot), xp = F x + u.
template <typename S, int N, int M>
__device__ __forceinline__ void t_predict(S* fr, const S* mf, const S* P, S* Pn) {
  using FF = FFrame<S, N, M>;
  using MF = ModelFrame<S, N, M>;
  constexpr int LD = FF::LD, LD2 = FF::LD2;
  const int ln = lane();
  const S* Fc = mf + MF::Fc;
  S* FPt = fr + FF::FPt;
  S* AUG2 = fr + FF::AUG2;
  {
    using P_ = Pick<N, N>;
    using TL = Tiling<N, N, P_::TM, P_::TN>;
    if (TL::active()) {
      const int r0 = TL::r0(), c0 = TL::c0();
      S acc[P_::TM][P_::TN];
      zero(acc);
      mma<N, P_::TM, P_::TN, 1, LD, LD, 1>(acc, Fc + r0, P + c0);
      put<P_::TM, P_::TN, 1, LD>(FPt + c0 * LD + r0, acc);
      put<P_::TM, P_::TN, LD2, 1>(AUG2 + r0 * LD2 + N + c0, acc);
    }
    if (ln < N)
      fr[FF::xp + ln] = mf[MF::u + ln] + matvec_row<N, N, 1, LD>(Fc, fr + FF::x, ln);
  }
  gsync();
  {
    using P_ = Pick<N, N>;
    using TL = Tiling<N, N, P_::TM, P_::TN>;
    if (TL::active()) {
      const int r0 = TL::r0(), c0 = TL::c0();
      S acc[P_::TM][P_::TN];
      init<P_::TM, P_::TN, LD, 1>(acc, mf + MF::Q + r0 * LD + c0);
      mma<N, P_::TM, P_::TN, 1, LD, LD, 1>(acc, FPt + r0, Fc + c0);
      put<P_::TM, P_::TN, LD, 1>(Pn + r0 * LD + c0, acc);  // symmetrised by the update
      put<P_::TM, P_::TN, LD2, 1>(AUG2 + r0 * LD2 + c0, acc);
    }
  }
  gsync();
}

// Smoothing element of step kp from its filtered (x, P) and the prediction
// (kalman_elems.hpp:151-193): E^T = PP^-1 FP, g = x - E xp, L = P - FP^T E^T
// (= P - E FP, symmetric); L overwrites P.  Stored to egl (E^T, g, L) and
// folded into the chunk element (E_a column-major in *Ea, g_a, L_a):
// E_a' = E_a E, g_a' = E_a g + g_a, L_a' = E_a L E_a^T + L_a.
template <typename S, int N, int M>
__device__ __forceinline__ void t_smooth_elem(S* fr, S*& P, S*& Ea, S* eglk, bool first,
                                              unsigned& e) {
  using FF = FFrame<S, N, M>;
  constexpr int LD = FF::LD, LD2 = FF::LD2;
  const int ln = lane();
  S* AUG2 = fr + FF::AUG2;
  S* FPt = fr + FF::FPt;
  S* La = fr + FF::La;
  gj_spd<N, 2 * N, LD2>(AUG2, fr + FF::pv, e);  // right half: E^T
  const S* Et = AUG2 + N;                        // E^T(r, c) at Et[r LD2 + c]
  {
    using P_ = Pick<N, N>;
    using TL = Tiling<N, N, P_::TM, P_::TN>;
    if (TL::active()) {
      const int r0 = TL::r0(), c0 = TL::c0();
      S acc[P_::TM][P_::TN];
      init<P_::TM, P_::TN, LD, 1>(acc, P + r0 * LD + c0);
      mma<N, P_::TM, P_::TN, LD, 1, LD2, 1, true>(acc, FPt + r0 * LD, Et + c0);
      put<P_::TM, P_::TN, LD, 1>(P + r0 * LD + c0, acc);
    }
    if (ln < N) {  // g = x - E xp
      S s = fr[FF::x + ln];
#pragma unroll
      for (int q = 0; q < N; ++q) s = sfma(-Et[q * LD2 + ln], fr[FF::xp + q], s);
      fr[FF::g + ln] = s;
    }
  }
  gsync();
  // per-step element to global: E^T, g, L (SOffs sizes)
  const SOffs SO(N);
  gstore_mat<N, LD2, false, false>(eglk + SO.E, Et);
  if (ln < N) eglk[SO.g + ln] = fr[FF::g + ln];
  gstore_mat<N, LD, false, false>(eglk + SO.L, P);
  if (first) {
    for (int i = ln; i < N * N; i += kGW) {
      const int r = i / N, c = i % N;
      Ea[r * LD + c] = Et[r * LD2 + c];  // E_a column-major = E^T row-major
      La[r * LD + c] = P[r * LD + c];
    }
    if (ln < N) fr[FF::ga + ln] = fr[FF::g + ln];
    gsync();
    return;
  }
  S* Tt = fr + FF::FPt;  // FP is dead: T = E_a L (column-major)
  {
    using P_ = Pick<N, N>;
    using TL = Tiling<N, N, P_::TM, P_::TN>;
    if (TL::active()) {
      const int r0 = TL::r0(), c0 = TL::c0();
      S acc[P_::TM][P_::TN];
      zero(acc);
      mma<N, P_::TM, P_::TN, 1, LD, LD, 1>(acc, Ea + r0, P + c0);
      put<P_::TM, P_::TN, 1, LD>(Tt + c0 * LD + r0, acc);
    }
    if (ln < N) {
      S s = fr[FF::ga + ln];
#pragma unroll
      for (int q = 0; q < N; ++q) s = sfma(Ea[q * LD + ln], fr[FF::g + q], s);
      fr[FF::ga + ln] = s;
    }
  }
  gsync();
  {
    using P_ = Pick<N, N>;
    using TL = Tiling<N, N, P_::TM, P_::TN>;
    if (TL::active()) {
      const int r0 = TL::r0(), c0 = TL::c0();
      S acc[P_::TM][P_::TN];
      // L_a += T E_a^T
      init<P_::TM, P_::TN, LD, 1>(acc, La + r0 * LD + c0);
      mma<N, P_::TM, P_::TN, 1, LD, LD, 1>(acc, Tt + r0, Ea + c0);
      put_sym<P_::TM, P_::TN, LD>(La, acc, r0, c0);
      // (E_a E)^T = E^T E_a^T (row-major = E_a' column-major) into the slot
      // of L, which the fold no longer reads
      zero(acc);
      mma<N, P_::TM, P_::TN, LD2, 1, LD, 1>(acc, Et + r0 * LD2, Ea + c0);
      put<P_::TM, P_::TN, LD, 1>(P + r0 * LD + c0, acc);
    }
  }
  {  // E_a moves to L's slot; the old E_a slot becomes free (the caller's P)
    S* t = Ea;
    Ea = P;
    P = t;
  }
  gsync();
}

// Kalman update of (x, P) with step-k measurement blocks (kalman_seq.hpp:58-99)
template <typename S, int N, int M>
__device__ __forceinline__ void t_update(S* fr, const S* mf, S* P, const S* y, unsigned& e) {
  using FF = FFrame<S, N, M>;
  using MF = ModelFrame<S, N, M>;
  constexpr int LD = FF::LD, LDP = FF::LDP, LDA3 = FF::LDA3, LDM = MF::LDM, LDR = MF::LDR;
  const int ln = lane();
  const S* Ht = mf + MF::Ht;
  S* HP = fr + FF::HP;
  S* AUG3 = fr + FF::AUG3;
  S* x = fr + FF::x;
  {  // HP = H P
    using P_ = Pick<M, N>;
    using TL = Tiling<M, N, P_::TM, P_::TN>;
    if (TL::active()) {
      const int r0 = TL::r0(), c0 = TL::c0();
      S acc[P_::TM][P_::TN];
      zero(acc);
      mma<N, P_::TM, P_::TN, 1, LDM, LD, 1>(acc, Ht + r0, P + c0);
      put<P_::TM, P_::TN, LDP, 1>(HP + r0 * LDP + c0, acc);
      put<P_::TM, P_::TN, LDA3, 1>(AUG3 + r0 * LDA3 + M + c0, acc);
    }
    if (ln < M) {
      const S v = y[ln] - mf[MF::d + ln] - matvec_row<M, N, 1, LDM>(Ht, x, ln);
      fr[FF::vv + ln] = v;
      AUG3[ln * LDA3 + M + N] = v;
    }
  }
  gsync();
  {  // S = HP H^T + R
    using P_ = Pick<M, M>;
    using TL = Tiling<M, M, P_::TM, P_::TN>;
    if (TL::active()) {
      const int r0 = TL::r0(), c0 = TL::c0();
      S acc[P_::TM][P_::TN];
      init<P_::TM, P_::TN, LDR, 1>(acc, mf + MF::R + r0 * LDR + c0);
      mma<N, P_::TM, P_::TN, LDP, 1, LDM, 1>(acc, HP + r0 * LDP, Ht + c0);
      put_sym<P_::TM, P_::TN, LDA3>(AUG3, acc, r0, c0);
    }
  }
  gsync();
  gj_spd<M, M + N + 1, LDA3>(AUG3, fr + FF::pv, e);  // [I | K^T | S^-1 v]
  {  // P -= K HP
    using P_ = Pick<N, N>;
    using TL = Tiling<N, N, P_::TM, P_::TN>;
    if (TL::active()) {
      const int r0 = TL::r0(), c0 = TL::c0();
      S acc[P_::TM][P_::TN];
      init<P_::TM, P_::TN, LD, 1>(acc, P + r0 * LD + c0);
      mma<M, P_::TM, P_::TN, 1, LDA3, LDP, 1, true>(acc, AUG3 + M + r0, HP + c0);
      put_sym<P_::TM, P_::TN, LD>(P, acc, r0, c0);
    }
    if (ln < N) {  // x += K v
      S s = x[ln];
#pragma unroll
      for (int q = 0; q < M; ++q) s = sfma(AUG3[q * LDA3 + M + ln], fr[FF::vv + q], s);
      x[ln] = s;
    }
  }
  gsync();
}

// finish: filter the chunk from the prefix of chunk c-1.  SMOOTH = false
// writes the filtered stats; SMOOTH = true the per-step smoothing elements
// and the chunk's smoother element (sagg, SOffs layout, E row-major).
template <typename S, int N, int M, bool SMOOTH>
__global__ void __launch_bounds__(kGW * kGroupsFinish)
    k_t_finish(ModelView<S> m, long long L, long long nchunks, const S* pre, S* mean, S* cov,
               S* sagg, S* egl, unsigned* err) {
  using FF = FFrame<S, N, M>;
  using MF = ModelFrame<S, N, M>;
  constexpr int LD = FF::LD;
  const bool inv = time_invariant(m);
  S *fr, *mf;
  frames<S, N, M, FF::size>(m, inv, fr, mf);
  const long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / kGW;
  if (c >= nchunks) return;
  const int ln = lane();
  unsigned e = 0;
  const long long k0 = c * L, k1 = min(k0 + L, m.t);
  const FOffs FO(N);
  const SOffs SO(N);
  S* P = fr + FF::P0;
  S* Pn = fr + FF::P1;
  S* Ea = fr + FF::Ea0;
  // incoming filtered state: the prior (chunk 0) or the prefix of chunk c-1
  {
    const S* xs = c == 0 ? m.m0 : pre + (c - 1) * FO.size + FO.b;
    const S* Ps = c == 0 ? m.p0 : pre + (c - 1) * FO.size + FO.C;
    sload_mat<N, LD, false>(P, Ps);
    if (ln < N) fr[FF::x + ln] = xs[ln];
  }
  gsync();
  for (long long k = k0; k < k1; ++k) {
    if (!inv) {
      load_model<S, N, M>(mf, m, k);
      gsync();
    }
    t_predict<S, N, M>(fr, mf, P, Pn);
    if constexpr (SMOOTH) {
      if (k > k0) t_smooth_elem<S, N, M>(fr, P, Ea, egl + (k - 1) * SO.size, k - 1 == k0, e);
    }
    {  // x = xp, P = PP
      S* t = P;
      P = Pn;
      Pn = t;
      if (ln < N) fr[FF::x + ln] = fr[FF::xp + ln];
    }
    gsync();
    const S* yk = inv ? m.Y(k) : mf + MF::y;
    t_update<S, N, M>(fr, mf, P, yk, e);
    if constexpr (!SMOOTH) {
      if (ln < N) mean[k * N + ln] = fr[FF::x + ln];
      gstore_mat<N, LD, false, true>(cov + k * N * N, P);
    }
  }
  if constexpr (SMOOTH) {  // element of the chunk's last step
    const long long kl = k1 - 1;
    const bool first = kl == k0;
    if (kl == m.last_step) {
      // a_T = (0, x_T, P_T) (kalman_elems.hpp:158-163)
      const SOffs SO2(N);
      S* eglk = egl + kl * SO2.size;
      for (int i = ln; i < N * N; i += kGW) eglk[SO2.E + i] = S(0);
      if (ln < N) eglk[SO2.g + ln] = fr[FF::x + ln];
      gstore_mat<N, LD, false, false>(eglk + SO2.L, P);
      S* La = fr + FF::La;
      if (first) {
        for (int i = ln; i < N * N; i += kGW) {
          const int r = i / N, cc = i % N;
          Ea[r * LD + cc] = S(0);
          La[r * LD + cc] = P[r * LD + cc];
        }
        if (ln < N) fr[FF::ga + ln] = fr[FF::x + ln];
      } else {
        // E_a' = 0, g_a' = E_a x + g_a, L_a' = E_a P E_a^T + L_a
        S* Tt = fr + FF::FPt;
        {
          using P_ = Pick<N, N>;
          using TL = Tiling<N, N, P_::TM, P_::TN>;
          if (TL::active()) {
            const int r0 = TL::r0(), c0 = TL::c0();
            S acc[P_::TM][P_::TN];
            zero(acc);
            mma<N, P_::TM, P_::TN, 1, LD, LD, 1>(acc, Ea + r0, P + c0);
            put<P_::TM, P_::TN, 1, LD>(Tt + c0 * LD + r0, acc);
          }
          if (ln < N) {
            S s = fr[FF::ga + ln];
#pragma unroll
            for (int q = 0; q < N; ++q) s = sfma(Ea[q * LD + ln], fr[FF::x + q], s);
            fr[FF::ga + ln] = s;
          }
        }
        gsync();
        {
          using P_ = Pick<N, N>;
          using TL = Tiling<N, N, P_::TM, P_::TN>;
          if (TL::active()) {
            const int r0 = TL::r0(), c0 = TL::c0();
            S acc[P_::TM][P_::TN];
            init<P_::TM, P_::TN, LD, 1>(acc, La + r0 * LD + c0);
            mma<N, P_::TM, P_::TN, 1, LD, LD, 1>(acc, Tt + r0, Ea + c0);
            put_sym<P_::TM, P_::TN, LD>(La, acc, r0, c0);
          }
        }
        gsync();
        for (int i = ln; i < N * N; i += kGW) Ea[(i / N) * LD + i % N] = S(0);
      }
      gsync();
    } else {
      if (!inv) {
        load_model<S, N, M>(mf, m, k1, true);
        gsync();
      }
      t_predict<S, N, M>(fr, mf, P, Pn);
      t_smooth_elem<S, N, M>(fr, P, Ea, egl + kl * SO.size, first, e);
    }
    S* o = sagg + c * SO.size;
    gstore_mat<N, LD, true, false>(o + SO.E, Ea);  // E_a row-major from column-major
    if (ln < N) o[SO.g + ln] = fr[FF::ga + ln];
    gstore_mat<N, LD, false, true>(o + SO.L, fr + FF::La);
  }
  if (e && ln == 0) atomicOr(err, e);
}

// smoother finish: backwards over the chunk from the suffix of chunk c+1,
// x_s(k) = E_k x_s(k+1) + g_k, P_s(k) = E_k P_s(k+1) E_k^T + L_k.
template <typename S, int N>
__global__ void __launch_bounds__(kGW * kGroupsSmooth)
    k_t_smoother_finish(long long T, long long L, long long nchunks, const S* suf,
                        const S* egl, S* mean, S* cov) {
  using SF = SFrame<S, N>;
  constexpr int LD = SF::LD;
  extern __shared__ __align__(16) unsigned char tsm[];
  S* fr = reinterpret_cast<S*>(tsm) + (threadIdx.x / kGW) * SF::size;
  const long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / kGW;
  if (c >= nchunks) return;
  const int ln = lane();
  const long long k0 = c * L, k1 = min(k0 + L, T);
  const SOffs SO(N);
  S* Ps = fr + SF::Ps;
  S* Tt = fr + SF::Tt;
  S* Et = fr + SF::Et;
  S* Lk = fr + SF::Lk;
  S* xs = fr + SF::xs;
  if (c + 1 < nchunks) {
    const S* s1 = suf + (c + 1) * SO.size;
    sload_mat<N, LD, false>(Ps, s1 + SO.L);
    if (ln < N) xs[ln] = s1[SO.g + ln];
  } else {  // the last step has E = 0: the incoming state is never used
    for (int i = ln; i < N * N; i += kGW) Ps[(i / N) * LD + i % N] = S(0);
    if (ln < N) xs[ln] = S(0);
  }
  for (long long i = k1 - 1; i >= k0; --i) {
    const S* ek = egl + i * SO.size;
    sload_mat<N, LD, false>(Et, ek + SO.E);
    sload_mat<N, LD, false>(Lk, ek + SO.L);
    if (ln < N) fr[SF::g + ln] = ek[SO.g + ln];
    gsync();
    {
      using P_ = Pick<N, N>;
      using TL = Tiling<N, N, P_::TM, P_::TN>;
      if (TL::active()) {  // T = E P_s (column-major)
        const int r0 = TL::r0(), c0 = TL::c0();
        S acc[P_::TM][P_::TN];
        zero(acc);
        mma<N, P_::TM, P_::TN, 1, LD, LD, 1>(acc, Et + r0, Ps + c0);
        put<P_::TM, P_::TN, 1, LD>(Tt + c0 * LD + r0, acc);
      }
      if (ln < N) {
        S s = fr[SF::g + ln];
#pragma unroll
        for (int q = 0; q < N; ++q) s = sfma(Et[q * LD + ln], xs[q], s);
        fr[SF::tmp + ln] = s;
      }
    }
    gsync();
    {
      using P_ = Pick<N, N>;
      using TL = Tiling<N, N, P_::TM, P_::TN>;
      if (TL::active()) {  // P_s = T E^T + L
        const int r0 = TL::r0(), c0 = TL::c0();
        S acc[P_::TM][P_::TN];
        init<P_::TM, P_::TN, LD, 1>(acc, Lk + r0 * LD + c0);
        mma<N, P_::TM, P_::TN, 1, LD, LD, 1>(acc, Tt + r0, Et + c0);
        put_sym<P_::TM, P_::TN, LD>(Ps, acc, r0, c0);
      }
      if (ln < N) xs[ln] = fr[SF::tmp + ln];
    }
    gsync();
    if (ln < N) mean[i * N + ln] = xs[ln];
    gstore_mat<N, LD, false, true>(cov + i * N * N, Ps);
  }
}

// ---- PTFS backward pass -------------------------------------------------------
template <typename S, int N, int M>
struct BFrame {  // backward finish
  static constexpr int V = vec16<S>();
  static constexpr int LD = ldpad<S>(N), MAT = N * LD;
  static constexpr int HAO = N + V, LDH = ldpad<S>(HAO + N), LDA = ldpad<S>(M + 2 * N + 1);
  static constexpr int LDG = ldpad<S>(2 * N + 1);  // [N | J A | w] and [M | P | rhs]
  static constexpr int J = 0, Aa = MAT, Ca = 2 * MAT + V, P = 3 * MAT + 2 * V,
                       Ja = 4 * MAT + 2 * V, HCA = 5 * MAT + 2 * V, AUG = HCA + M * LDH,
                       G = AUG + M * LDA,
                       eta = G + N * LDG, etaa = eta + up16<S>(N), ba = etaa + up16<S>(N),
                       x = ba + up16<S>(N), vv = x + up16<S>(N), pv = vv + up16<S>(M),
                       size = pv + 2 * up16<S>(N > M ? N : M);
};
constexpr int kGroupsBwd = 4;

// The backward pass of the two-filter smoother (Alg. 7, kalman_par.hpp:
// 183-238) for chunk c, walking its slots backwards: slot i holds the filter
// element of step i+1 (`ms` is the model shifted by one step; no element past
// the series' last transition, build_shifted_filter_elems kalman_par.hpp:
// 63-89).  The running backward information (eta, J) starts from the
// reverse-scanned suffix of chunk c+1; at each slot it becomes the eta / J
// rows of a (x) (eta, J) (Lemma 1, kalman_elems.hpp:267-336, with the element
// built from the identity by the conditional-Kalman update), then the
// two-filter combination (kalman_seq.hpp:239-260) turns the filtered (x, P)
// of step i -- read from mean / cov -- into the smoothed stats, written in
// place.  Both non-symmetric solves are pivoted Gauss-Jordan eliminations.
template <typename S, int N, int M>
__global__ void __launch_bounds__(kGW * kGroupsBwd)
    k_t_bwd_finish(ModelView<S> ms, long long T, long long L, long long nchunks, const S* suf,
                   S* mean, S* cov, unsigned* err) {
  using BF = BFrame<S, N, M>;
  using MF = ModelFrame<S, N, M>;
  constexpr int LD = BF::LD, LDH = BF::LDH, LDA = BF::LDA, LDG = BF::LDG, LDM = MF::LDM,
                LDR = MF::LDR;
  const bool inv = time_invariant(ms);
  S *fr, *mf;
  frames<S, N, M, BF::size>(ms, inv, fr, mf);
  const long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / kGW;
  if (c >= nchunks) return;
  const int ln = lane();
  unsigned e = 0;
  const long long k0 = c * L, k1 = min(k0 + L, T);
  const FOffs FO(N);
  S* J = fr + BF::J;
  S* Aa = fr + BF::Aa;
  S* Ca = fr + BF::Ca;
  S* P = fr + BF::P;
  S* Ja = fr + BF::Ja;
  S* HCA = fr + BF::HCA;
  S* AUG = fr + BF::AUG;
  S* G = fr + BF::G;
  S* eta = fr + BF::eta;
  S* etaa = fr + BF::etaa;
  S* ba = fr + BF::ba;
  S* x = fr + BF::x;
  S* vv = fr + BF::vv;
  S* pv = fr + BF::pv;
  const S* Fc = mf + MF::Fc;
  const S* Qm = mf + MF::Q;
  const S* Ht = mf + MF::Ht;
  const S* Rm = mf + MF::R;
  if (c + 1 < nchunks) {  // the suffix of the later chunks
    const S* s1 = suf + (c + 1) * FO.size;
    sload_mat<N, LD, false>(J, s1 + FO.J);
    if (ln < N) eta[ln] = s1[FO.eta + ln];
  } else {
    for (int i = ln; i < N * N; i += kGW) J[(i / N) * LD + i % N] = S(0);
    if (ln < N) eta[ln] = S(0);
  }
  gsync();
  // A time-invariant model has the same element matrices (A_a, C_a, J_a and
  // the gain) at every slot; only b_a and eta_a follow y.  They are built
  // once per chunk, and each slot then costs three matrix-vector products.
  bool built = false;
  for (long long i = k1 - 1; i >= k0; --i) {
    if (i < ms.t && inv && built) {
      if (ln < M) {  // v = y - H u - d
        const S v = ms.Y(i)[ln] - mf[MF::d + ln] - matvec_row<M, N, 1, LDM>(Ht, mf + MF::u, ln);
        vv[ln] = v;
      }
      gsync();
      if (ln < N) {  // b_a = u + K v, eta_a = (S^-1 HA)^T v
        S b = mf[MF::u + ln], h = S(0);
#pragma unroll
        for (int q = 0; q < M; ++q) {
          b = sfma(AUG[q * LDA + M + ln], vv[q], b);
          h = sfma(AUG[q * LDA + M + N + ln], vv[q], h);
        }
        ba[ln] = b;
        etaa[ln] = h;
      }
      gsync();
    } else if (i < ms.t) {  // slot i holds the element of step i+1
      if (!inv) {
        load_model<S, N, M>(mf, ms, i);
        gsync();
      }
      built = true;
      // the element from the identity: A = F, b = u, C = Q, updated with y
      {  // [HC | HA] = H [Q | F]
        using P_ = Pick<M, 2 * N>;
        using TL = Tiling<M, 2 * N, P_::TM, P_::TN>;
        if (TL::active()) {
          const int r0 = TL::r0(), c0 = TL::c0();
          S acc[P_::TM][P_::TN];
          zero(acc);
          if (c0 < N)
            mma<N, P_::TM, P_::TN, 1, LDM, LD, 1>(acc, Ht + r0, Qm + c0);
          else  // F(k, c) = Fc[c LD + k]
            mma<N, P_::TM, P_::TN, 1, LDM, 1, LD>(acc, Ht + r0, Fc + (c0 - N) * LD);
          put<P_::TM, P_::TN, LDH, 1>(HCA + r0 * LDH + (c0 < N ? c0 : c0 - N + BF::HAO), acc);
          put<P_::TM, P_::TN, LDA, 1>(AUG + r0 * LDA + M + c0, acc);
        }
        if (ln < M) {  // v = y - H u - d
          const S y = inv ? ms.Y(i)[ln] : mf[MF::y + ln];
          const S v = y - mf[MF::d + ln] - matvec_row<M, N, 1, LDM>(Ht, mf + MF::u, ln);
          vv[ln] = v;
          AUG[ln * LDA + M + 2 * N] = v;
        }
      }
      gsync();
      {  // S = HC H^T + R
        using P_ = Pick<M, M>;
        using TL = Tiling<M, M, P_::TM, P_::TN>;
        if (TL::active()) {
          const int r0 = TL::r0(), c0 = TL::c0();
          S acc[P_::TM][P_::TN];
          init<P_::TM, P_::TN, LDR, 1>(acc, Rm + r0 * LDR + c0);
          mma<N, P_::TM, P_::TN, LDH, 1, LDM, 1>(acc, HCA + r0 * LDH, Ht + c0);
          put_sym<P_::TM, P_::TN, LDA>(AUG, acc, r0, c0);
        }
      }
      gsync();
      gj_spd<M, M + 2 * N + 1, LDA>(AUG, pv, e);  // [I | K^T | S^-1 HA | S^-1 v]
      {  // J_a = HA^T S^-1 HA
        using P_ = Pick<N, N>;
        using TL = Tiling<N, N, P_::TM, P_::TN>;
        if (TL::active()) {
          const int r0 = TL::r0(), c0 = TL::c0();
          S acc[P_::TM][P_::TN];
          zero(acc);
          mma<M, P_::TM, P_::TN, 1, LDH, LDA, 1>(acc, HCA + BF::HAO + r0, AUG + M + N + c0);
          put_sym<P_::TM, P_::TN, LD>(Ja, acc, r0, c0);
        }
      }
      {  // [A_a | C_a] = [F | Q] - K [HA | HC]
        using P_ = Pick<N, 2 * N>;
        using TL = Tiling<N, 2 * N, P_::TM, P_::TN>;
        if (TL::active()) {
          const int r0 = TL::r0(), c0 = TL::c0();
          S acc[P_::TM][P_::TN];
          const bool left = c0 < N;
          if (left)
            init<P_::TM, P_::TN, 1, LD>(acc, Fc + c0 * LD + r0);  // F(r, c) = Fc[c LD + r]
          else
            init<P_::TM, P_::TN, LD, 1>(acc, Qm + r0 * LD + (c0 - N));
          const S* rp = left ? HCA + BF::HAO + c0 : HCA + (c0 - N);
          mma<M, P_::TM, P_::TN, 1, LDA, LDH, 1, true>(acc, AUG + M + r0, rp);
          if (left)
            put<P_::TM, P_::TN, LD, 1>(Aa + r0 * LD + c0, acc);
          else
            put_sym<P_::TM, P_::TN, LD>(Ca, acc, r0, c0 - N);
        }
      }
      if (ln < N) {  // b_a = u + K v, eta_a = HA^T S^-1 v
        S b = mf[MF::u + ln], h = S(0);
#pragma unroll
        for (int q = 0; q < M; ++q) {
          b = sfma(AUG[q * LDA + M + ln], vv[q], b);
          h = sfma(HCA[q * LDH + BF::HAO + ln], AUG[q * LDA + M + 2 * N], h);
        }
        ba[ln] = b;
        etaa[ln] = h;
      }
      gsync();
    }
    if (i < ms.t) {
      // (eta, J) <- a (x) (eta, J): G = [I + J C_a | J A_a | eta - J b_a]
      {
        using P_ = Pick<N, 2 * N>;
        using TL = Tiling<N, 2 * N, P_::TM, P_::TN>;
        if (TL::active()) {
          const int r0 = TL::r0(), c0 = TL::c0();
          S acc[P_::TM][P_::TN];
          zero(acc);
          const bool left = c0 < N;
          mma<N, P_::TM, P_::TN, 1, LD, LD, 1>(acc, J + r0, left ? Ca + c0 : Aa + (c0 - N));
          if (left) {
#pragma unroll
            for (int a = 0; a < P_::TM; ++a)
#pragma unroll
              for (int b = 0; b < P_::TN; ++b)
                if (r0 + a == c0 + b) acc[a][b] += S(1);
          }
          put<P_::TM, P_::TN, LDG, 1>(G + r0 * LDG + c0, acc);
        }
        if (ln < N) {
          S w = eta[ln];
#pragma unroll
          for (int q = 0; q < N; ++q) w = sfma(-J[ln * LD + q], ba[q], w);
          G[ln * LDG + 2 * N] = w;
        }
      }
      gsync();
      gj_piv<N, 2 * N + 1, LDG>(G, pv, e);  // [I | N^-1 J A_a | N^-1 w]
      {  // J = A_a^T (N^-1 J A_a) + J_a ; eta = A_a^T N^-1 w + eta_a
        using P_ = Pick<N, N>;
        using TL = Tiling<N, N, P_::TM, P_::TN>;
        if (TL::active()) {
          const int r0 = TL::r0(), c0 = TL::c0();
          S acc[P_::TM][P_::TN];
          init<P_::TM, P_::TN, LD, 1>(acc, Ja + r0 * LD + c0);
          mma<N, P_::TM, P_::TN, 1, LD, LDG, 1>(acc, Aa + r0, G + N + c0);
          put_sym<P_::TM, P_::TN, LD>(J, acc, r0, c0);
        }
        if (ln < N) {
          S h = etaa[ln];
#pragma unroll
          for (int q = 0; q < N; ++q) h = sfma(Aa[q * LD + ln], G[q * LDG + 2 * N], h);
          eta[ln] = h;
        }
      }
      gsync();
    }
    // two-filter combination with the filtered (x, P) of step i
    sload_mat<N, LD, false>(P, cov + i * N * N);
    if (ln < N) x[ln] = mean[i * N + ln];
    gsync();
    {  // G = [I + P J | P | x + P eta]
      using P_ = Pick<N, N>;
      using TL = Tiling<N, N, P_::TM, P_::TN>;
      if (TL::active()) {
        const int r0 = TL::r0(), c0 = TL::c0();
        S acc[P_::TM][P_::TN];
        zero(acc);
        mma<N, P_::TM, P_::TN, 1, LD, LD, 1>(acc, P + r0, J + c0);
#pragma unroll
        for (int a = 0; a < P_::TM; ++a)
#pragma unroll
          for (int b = 0; b < P_::TN; ++b)
            if (r0 + a == c0 + b) acc[a][b] += S(1);
        put<P_::TM, P_::TN, LDG, 1>(G + r0 * LDG + c0, acc);
      }
      if (ln < N) {
        S r = x[ln];
#pragma unroll
        for (int q = 0; q < N; ++q) r = sfma(P[ln * LD + q], eta[q], r);
        G[ln * LDG + 2 * N] = r;
      }
      for (int k = ln; k < N * N; k += kGW) G[(k / N) * LDG + N + k % N] = P[(k / N) * LD + k % N];
    }
    gsync();
    gj_piv<N, 2 * N + 1, LDG>(G, pv, e);  // [I | P_s | x_s]
    if (ln < N) mean[i * N + ln] = G[ln * LDG + 2 * N];
    gstore_mat<N, LDG, false, true>(cov + i * N * N, G + N);
    gsync();
  }
  if (e && ln == 0) atomicOr(err, e);
}

// ---- host dispatch --------------------------------------------------------------
template <typename S, int N, int M>
int tile_run_t(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a, S* mean, S* cov,
               void* (*alloc)(size_t, void*), void* actx) {
  using namespace wide;
  const long long T = m.t;
  if (T == 0) return 0;
  const bool inv = time_invariant(m);
  const int smem_r = cta_smem<S, N, M, RFrame<S, N, M>::size, kGroupsReduce>(inv);
  const int smem_f = cta_smem<S, N, M, FFrame<S, N, M>::size, kGroupsFinish>(inv);
  const int smem_s = (int)sizeof(S) * kGroupsSmooth * SFrame<S, N>::size;
  long long Lc = a.chunk;
  // auto: `waves` waves of co-resident finish groups, default ONE for PKF /
  // PRTS -- a longer chunk amortises the per-chunk reduce and the scan, and
  // the batch path's concurrent series fill the machine anyway
  // (tools/config5.py --waves, f64 19.10 / 19.64 / 20.78 ms per series at
  // 1 / 2 / 4 waves, batch 64) -- and FOUR for PTFS, whose backward finish
  // holds fewer groups per SM (f64 60.7 / 51.3 / 51.5 / 54.3 ms per series at
  // 1 / 2 / 4 / 8 waves, f32 28.4 / 24.5 / 23.0 / 24.3; 3 waves: 56.7 f64)
  if (Lc < 1) {
    const int per_sm = kernel_setup(k_t_finish<S, N, M, true>, kGW * kGroupsFinish, smem_f);
    const long long resident = (long long)device_sms() * (per_sm > 0 ? per_sm : 1) *
                               kGroupsFinish * (a.waves > 0 ? a.waves : (a.method == 2 ? 4 : 1));
    Lc = (T + resident - 1) / resident;
    if (Lc < 1) Lc = 1;
    if (a.alg == 0 && Lc < seq_chunk_floor(T)) Lc = seq_chunk_floor(T);
  }
  const long long nch = (T + Lc - 1) / Lc;
  const int alg = a.alg == 6 ? 3 : a.alg;
  const long long npad = alg == 0 ? nch : (long long)next_pow2(nch);
  ScanPlan plan;
  if (npad > 1) {
    plan = make_scan_plan(alg, a.sengupta_n, npad);
    if (plan.status) return plan.status;
  }
  const FOffs FO(N);
  const SOffs SO(N);
  S* agg = (S*)alloc(sizeof(S) * FO.size * npad, actx);
  S* aux1 = (S*)alloc(sizeof(S) * FO.size * (plan.cap1 ? plan.cap1 : 1), actx);
  S* aux2 = (S*)alloc(sizeof(S) * FO.size * (plan.cap2 ? plan.cap2 : 1), actx);
  S* sagg = a.method == 1 ? (S*)alloc(sizeof(S) * SO.size * npad, actx) : nullptr;
  S* egl = a.method == 1 ? (S*)alloc(sizeof(S) * SO.size * T, actx) : nullptr;
  if (!agg || !aux1 || !aux2 || (a.method == 1 && (!sagg || !egl))) return 8;
  auto grid = [&](int g) { return wide_blocks(nch, g); };
  WideFilterOps<S> fops{L.err, N};
  WideSmootherOps<S> sops{N};
  constexpr int br = kGW * kGroupsReduce, bf = kGW * kGroupsFinish, bs = kGW * kGroupsSmooth;
  kernel_setup(k_t_reduce<S, N, M>, br, smem_r);
  k_t_reduce<S, N, M><<<grid(kGroupsReduce), br, smem_r, L.stream>>>(m, Lc, nch, agg, L.err);
  L.count("tile_filter_reduce");
  if (npad > nch) {
    k_wide_fill_identity<<<wide_blocks(npad - nch, 4), 128, 0, L.stream>>>(
        fops, ElemBuf<S>{agg, npad, npad, 0}, nch, npad);
    L.count("fill_identity");
  }
  if (npad > 1) wide_scan(L, fops, agg, npad, aux1, aux2, plan, 0);
  if (a.method == 0 || a.method == 2) {
    kernel_setup(k_t_finish<S, N, M, false>, bf, smem_f);
    k_t_finish<S, N, M, false><<<grid(kGroupsFinish), bf, smem_f, L.stream>>>(
        m, Lc, nch, agg, mean, cov, nullptr, nullptr, L.err);
    L.count("tile_filter_finish");
    if (a.method == 0) return 0;
    // PTFS backward pass: shifted elements (slot i = step i+1) reduced per
    // chunk from the identity, reverse scan, backward finish fused with the
    // two-filter combination over the filtered stats in mean / cov
    ModelView<S> ms = m;
    ms.f += m.sf; ms.u += m.su; ms.q += m.sq; ms.h += m.sh; ms.d += m.sd; ms.r += m.sr;
    ms.y += m.sy;
    ms.t = T - 1;
    ms.prior_first = 0;
    ms.last_step = ms.t - 1;
    const long long nch_s = ms.t > 0 ? (ms.t + Lc - 1) / Lc : 0;
    if (nch_s > 0) {
      k_t_reduce<S, N, M><<<wide_blocks(nch_s, kGroupsReduce), br, smem_r, L.stream>>>(
          ms, Lc, nch_s, agg, L.err);
      L.count("tile_bwd_reduce");
    }
    if (npad > nch_s) {
      k_wide_fill_identity<<<wide_blocks(npad - nch_s, 4), 128, 0, L.stream>>>(
          fops, ElemBuf<S>{agg, npad, npad, 0}, nch_s, npad);
      L.count("fill_identity");
    }
    if (npad > 1) wide_scan(L, fops, agg, npad, aux1, aux2, plan, 1);
    const int smem_b = cta_smem<S, N, M, BFrame<S, N, M>::size, kGroupsBwd>(inv);
    constexpr int bb = kGW * kGroupsBwd;
    kernel_setup(k_t_bwd_finish<S, N, M>, bb, smem_b);
    k_t_bwd_finish<S, N, M><<<grid(kGroupsBwd), bb, smem_b, L.stream>>>(ms, T, Lc, nch, agg, mean,
                                                                     cov, L.err);
    L.count("tile_bwd_finish_tf_combine");
    return 0;
  }
  kernel_setup(k_t_finish<S, N, M, true>, bf, smem_f);
  k_t_finish<S, N, M, true><<<grid(kGroupsFinish), bf, smem_f, L.stream>>>(
      m, Lc, nch, agg, mean, cov, sagg, egl, L.err);
  L.count("tile_filter_finish_smoother_reduce");
  if (npad > nch) {
    k_wide_fill_identity<<<wide_blocks(npad - nch, 4), 128, 0, L.stream>>>(
        sops, ElemBuf<S>{sagg, npad, npad, 0}, nch, npad);
    L.count("fill_identity");
  }
  if (npad > 1) wide_scan(L, sops, sagg, npad, aux1, aux2, plan, 1);
  kernel_setup(k_t_smoother_finish<S, N>, bs, smem_s);
  k_t_smoother_finish<S, N><<<grid(kGroupsSmooth), bs, smem_s, L.stream>>>(T, Lc, nch, sagg, egl,
                                                                          mean, cov);
  L.count("tile_smoother_finish");
  return 0;
}

// (nx, ny) with a register-tiled instantiation; -1 otherwise
#define PSK_TILE_DIMS(X) X(16, 8)

template <typename S>
int tile_run(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a, S* mean, S* cov,
             void* (*alloc)(size_t, void*), void* actx) {
  if (!m.prior_first || m.last_step != m.t - 1) return -1;
#define PSK_CASE(A, B) \
  if (m.nx == A && m.ny == B) return tile_run_t<S, A, B>(L, m, a, mean, cov, alloc, actx);
  PSK_TILE_DIMS(PSK_CASE)
#undef PSK_CASE
  return -1;
}

}  // namespace tile
}  // namespace psk
