// psk_fast_impl.cuh -- host dispatch of the fast (chunked) path and its template
// instantiations.  See psk_fast.cuh for the formulation.
#pragma once
#include <cuda_runtime.h>

#include "psk_dlb.cuh"
#include "psk_exact.h"
#include "psk_fast.cuh"
#include "psk_levels.cuh"

namespace psk {

namespace {
inline int blocks_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  return (int)(g < 1 ? 1 : g);
}
inline int grid_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148LL * 64) g = 148LL * 64;
  return (int)g;
}
constexpr int kBlock = 128;
}  // namespace

// Scan of chunk elements: level-by-level plan (alg 0..5) or the single-pass
// decoupled look-back (alg 6).  `buf` holds npad slots (identity padded).
template <class Ops>
static int chunk_scan(ExactLaunch& L, const Ops& ops, const FastArgs& a,
                      typename Ops::S* buf, long long nchunks, long long npad,
                      int rev, typename Ops::S* aux1, typename Ops::S* aux2,
                      const ScanPlan& plan, void* dlb_state) {
  using S = typename Ops::S;
  if (a.alg == 6) {
    dlb_scan<Ops>(L, ops, buf, nchunks, rev, aux1, dlb_state);
    return 0;
  }
  Bufs3<Ops> bufs;
  bufs.b[0] = ElemBuf<S>{buf, npad, npad, rev};
  bufs.b[1] = ElemBuf<S>{aux1, plan.cap1 ? plan.cap1 : 1, plan.cap1, rev};
  bufs.b[2] = ElemBuf<S>{aux2, plan.cap2 ? plan.cap2 : 1, plan.cap2, rev};
  for (const LevelDesc& d : plan.levels) {
    const int g = d.kind == kLvSeqChain ? 1 : grid_for(d.count, kBlock);
    k_level<Ops><<<g, kBlock, 0, L.stream>>>(ops, bufs, d);
    L.count("chunk_scan_level");
  }
  return 0;
}

template <typename S, int NX, int NY>
static int fast_run_t(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a,
                      S* mean, S* cov, void* (*alloc)(size_t, void*),
                      void* actx) {
  const long long T = m.t;
  if (T == 0) return 0;
  const long long Lc = a.chunk < 1 ? 1 : a.chunk;
  const long long nchunks = (T + Lc - 1) / Lc;
  const bool dlb = a.alg == 6;
  const long long npad =
      (dlb || a.alg == 0) ? nchunks : (long long)next_pow2(nchunks);
  ScanPlan plan;
  if (!dlb) {
    plan = make_scan_plan(a.alg, a.sengupta_n, npad);
    if (plan.status) return plan.status;
  }
  constexpr int FS = FLayout<NX>::size;
  const long long aux1n = dlb ? 0 : plan.cap1, aux2n = dlb ? 0 : plan.cap2;
  S* agg = (S*)alloc(sizeof(S) * FS * npad, actx);
  S* aux1 = (S*)alloc(sizeof(S) * FS * (aux1n ? aux1n : 1), actx);
  S* aux2 = (S*)alloc(sizeof(S) * FS * (aux2n ? aux2n : 1), actx);
  void* dlb_state = dlb ? alloc(dlb_state_bytes<S, NX>(nchunks), actx) : nullptr;
  if (!agg || !aux1 || !aux2 || (dlb && !dlb_state)) return 8;

  FastFilterOps<S, NX> fops{L.err};
  FastSmootherOps<S, NX> sops{L.err};
  const int g = blocks_for(nchunks, kBlock);

  // ---- forward filter (PKF; first half of PRTS / PTFS) ----
  k_filter_reduce<S, NX, NY><<<g, kBlock, 0, L.stream>>>(m, Lc, nchunks, agg, npad, L.err);
  L.count("filter_reduce");
  if (npad > nchunks) {
    k_fill_identity<<<blocks_for(npad - nchunks, kBlock), kBlock, 0, L.stream>>>(
        fops, ElemBuf<S>{agg, npad, npad, 0}, nchunks, npad);
    L.count("fill_identity");
  }
  chunk_scan(L, fops, a, agg, nchunks, npad, 0, aux1, aux2, plan, dlb_state);
  k_filter_finish<S, NX, NY><<<g, kBlock, 0, L.stream>>>(m, Lc, nchunks, agg, npad, mean, cov, L.err);
  L.count("filter_finish");

  if (a.method == 1) {  // ---- RTS smoother ----
    k_smoother_reduce<S, NX><<<g, kBlock, 0, L.stream>>>(m, mean, cov, Lc, nchunks, agg, npad, L.err);
    L.count("smoother_reduce");
    if (npad > nchunks) {
      k_fill_identity<<<blocks_for(npad - nchunks, kBlock), kBlock, 0, L.stream>>>(
          sops, ElemBuf<S>{agg, npad, npad, 0}, nchunks, npad);
      L.count("fill_identity");
    }
    chunk_scan(L, sops, a, agg, nchunks, npad, 1, aux1, aux2, plan, dlb_state);
    k_smoother_finish<S, NX><<<g, kBlock, 0, L.stream>>>(m, Lc, nchunks, agg, npad, mean, cov, L.err);
    L.count("smoother_finish");
  } else if (a.method == 2) {  // ---- two-filter smoother ----
    k_bwd_reduce<S, NX, NY><<<g, kBlock, 0, L.stream>>>(m, Lc, nchunks, agg, npad, L.err);
    L.count("bwd_reduce");
    if (npad > nchunks) {
      k_fill_identity<<<blocks_for(npad - nchunks, kBlock), kBlock, 0, L.stream>>>(
          fops, ElemBuf<S>{agg, npad, npad, 0}, nchunks, npad);
      L.count("fill_identity");
    }
    chunk_scan(L, fops, a, agg, nchunks, npad, 1, aux1, aux2, plan, dlb_state);
    k_bwd_finish<S, NX, NY><<<g, kBlock, 0, L.stream>>>(m, Lc, nchunks, agg, npad, mean, cov, L.err);
    L.count("bwd_finish_tf_combine");
  }
  return 0;
}

// compiled (nx, ny) instantiations of the fast path
#define PSK_FAST_DIMS(X) \
  X(1, 1)                \
  X(2, 1)                \
  X(2, 2)                \
  X(3, 1)                \
  X(3, 2)                \
  X(3, 3)                \
  X(4, 1)                \
  X(4, 2)                \
  X(4, 3)                \
  X(4, 4)

template <typename S>
bool fast_supported(int nx, int ny) {
#define PSK_CASE(A, B) \
  if (nx == A && ny == B) return true;
  PSK_FAST_DIMS(PSK_CASE)
#undef PSK_CASE
  return false;
}

template <typename S>
int fast_run(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a,
             S* mean, S* cov, void* (*alloc)(size_t, void*), void* actx) {
#define PSK_CASE(A, B) \
  if (m.nx == A && m.ny == B) return fast_run_t<S, A, B>(L, m, a, mean, cov, alloc, actx);
  PSK_FAST_DIMS(PSK_CASE)
#undef PSK_CASE
  return -1;
}

}  // namespace psk
