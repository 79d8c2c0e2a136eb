// psk_fast_impl.cuh -- host dispatch of the fast (chunked) path, split into
// phases so that a time-sharded run (distributed.py) can exchange shard
// aggregates between the reduce+scan and the finish of each pass.
#pragma once
#include <cuda_runtime.h>

#include "psk_dlb.cuh"
#include "psk_exact.h"
#include "psk_fast.cuh"
#include "psk_levels.cuh"
#include "psk_tiles.cuh"
#include "psk_tma.hpp"

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

// Let device `dev` read / copy from `peer` over NVLink when the pair supports
// it (idempotent; the copy falls back to staging through the host otherwise).
inline void enable_peer(int dev, int peer) {
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, dev, peer) != cudaSuccess || !can) return;
  int cur = -1;
  cudaGetDevice(&cur);
  cudaSetDevice(dev);
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();  // clear the sticky-free error
  cudaSetDevice(cur);
}

// The model shifted by one step (step i of the view = step i + 1 of m,
// t - 1 steps, no prior): the backward pass of PTFS walks the elements
// a(step i+1) at slot i.
template <typename S>
ModelView<S> shift_model(const ModelView<S>& m) {
  ModelView<S> v = m;
  v.f += m.sf;
  v.u += m.su;
  v.q += m.sq;
  v.h += m.sh;
  v.d += m.sd;
  v.r += m.sr;
  v.y += m.sy;
  // a time shard that does not end the series carries one extra step of
  // every field (last_step < 0), so its shifted view keeps all t slots
  v.t = m.last_step < 0 ? m.t : (m.t > 0 ? m.t - 1 : 0);
  v.prior_first = 0;
  v.last_step = v.t - 1;
  return v;
}

// Recursive tile sweep (psk_tiles.cuh) of the view `v` of buffer `a`.
template <class Ops>
static void tiled_sweep(ExactLaunch& L, const Ops& ops, const ElemBuf<typename Ops::S>& a,
                        const ElemBuf<typename Ops::S>& orig, TileView v, bool blelloch,
                        bool outer) {
  using S = typename Ops::S;
  const int smem = (int)(sizeof(S) * Ops::kSize * kTileSlots);
  const ElemBuf<S> none{nullptr, 1, 0, a.rev};
  const ElemBuf<S> og = outer ? orig : none;
  if (v.n <= kTile) {
    if (blelloch) {
      kernel_setup(k_tile_all<Ops, true>, kTile, smem);
      k_tile_all<Ops, true><<<1, kTile, smem, L.stream>>>(ops, a, og, v, og);
    } else {
      kernel_setup(k_tile_all<Ops, false>, kTile, smem);
      k_tile_all<Ops, false><<<1, kTile, smem, L.stream>>>(ops, a, none, v, none);
    }
    L.count("chunk_scan_tile_all");
    return;
  }
  const int grid = (int)(v.n / kTile);
  kernel_setup(k_tile_up<Ops>, kTile, smem);
  k_tile_up<Ops><<<grid, kTile, smem, L.stream>>>(ops, a, og, v, none, ArenaOut{});
  L.count("chunk_scan_tile_up");
  tiled_sweep(L, ops, a, orig, TileView{v.n / kTile, v.stride * kTile,
                                        v.off + (kTile - 1) * v.stride},
              blelloch, false);
  if (blelloch) {
    kernel_setup(k_tile_down<Ops, true>, kTile, smem);
    k_tile_down<Ops, true><<<grid, kTile, smem, L.stream>>>(ops, a, og, v, none, 0);
  } else {
    kernel_setup(k_tile_down<Ops, false>, kTile, smem);
    k_tile_down<Ops, false><<<grid, kTile, smem, L.stream>>>(ops, a, none, v, none, 0);
  }
  L.count("chunk_scan_tile_down");
}

// Scan of chunk elements: level-by-level plan (alg 0..5) or the single-pass
// decoupled look-back (alg 6).  `buf` holds npad slots (identity padded).
template <class Ops>
static void chunk_scan(ExactLaunch& L, const Ops& ops, const FastArgs& a,
                       typename Ops::S* buf, long long nchunks, long long npad,
                       int rev, typename Ops::S* aux1, typename Ops::S* aux2,
                       const ScanPlan& plan, void* dlb_state, long long cap = 0) {
  using S = typename Ops::S;
  if (a.alg == 6) {  // buf in ChunkOrder{nchunks, dlb_per<Ops>, rev} (FastScratch)
    dlb_scan<Ops>(L, ops, buf, nchunks, cap, rev, 1, dlb_state);
    return;
  }
  Bufs3<Ops> bufs;
  bufs.b[0] = ElemBuf<S>{buf, npad, npad, rev};
  bufs.b[1] = ElemBuf<S>{aux1, plan.cap1 ? plan.cap1 : 1, plan.cap1, rev};
  bufs.b[2] = ElemBuf<S>{aux2, plan.cap2 ? plan.cap2 : 1, plan.cap2, rev};
  if ((a.alg == 2 || a.alg == 3) && npad >= 2) {
    // Blelloch / Ladner-Fischer as shared-memory tile sweeps (psk_tiles.cuh)
    tiled_sweep(L, ops, bufs.b[0], a.alg == 2 ? bufs.b[1] : ElemBuf<S>{nullptr, 1, 0, rev},
                TileView{npad, 1, 0}, a.alg == 2, true);
    return;
  }
  // Sengupta hybrid: the reduce passes d <= log2(tile) and the distribute
  // passes d < log2(tile) run as tile sweeps; the rest level by level
  int sg_levels = 0;  // number of reduce passes (dstar)
  for (const LevelDesc& d : plan.levels) sg_levels += d.kind == kLvSgReduce;
  const int tl = (int)log2_exact(kTile);
  const bool sg_tiled = (a.alg == 4 || a.alg == 5) && sg_levels >= tl;
  const int smem = (int)(sizeof(S) * Ops::kSize * kTileSlots);
  const ElemBuf<S> none{nullptr, 1, 0, rev};
  int reduce_seen = 0;
  long long root_off = 0;
  bool dist_tail = false;
  for (const LevelDesc& d : plan.levels) {
    if (sg_tiled && d.kind == kLvSgReduce) {
      ++reduce_seen;  // level reduce_seen, arena offset d.p0
      if (reduce_seen < tl) continue;
      if (reduce_seen == tl) {
        ArenaOut ao{};
        // offsets of arena levels 1..tl (the plan's reduce passes, in order)
        int q = 0;
        for (const LevelDesc& e : plan.levels)
          if (e.kind == kLvSgReduce && q < tl) ao.off[++q] = e.p0;
        root_off = ao.off[tl];
        kernel_setup(k_tile_up<Ops>, kTile, smem);
        k_tile_up<Ops><<<(int)(npad / kTile), kTile, smem, L.stream>>>(
            ops, bufs.b[0], none, TileView{npad, 1, 0}, bufs.b[1], ao);
        L.count("chunk_scan_tile_up");
        continue;
      }
    }
    if (sg_tiled && d.kind == kLvSgDist && d.count > npad / kTile) {
      dist_tail = true;  // distribute passes below the tile roots: fused
      continue;
    }
    const int g = d.kind == kLvSeqChain ? 1 : grid_for(d.count, kBlock);
    k_level<Ops><<<g, kBlock, 0, L.stream>>>(ops, bufs, d);
    L.count("chunk_scan_level");
  }
  if (dist_tail) {
    kernel_setup(k_tile_down<Ops, false>, kTile, smem);
    k_tile_down<Ops, false><<<(int)(npad / kTile), kTile, smem, L.stream>>>(
        ops, bufs.b[0], none, TileView{npad, 1, 0}, bufs.b[1], root_off);
    L.count("chunk_scan_tile_down");
  }
}

// Automatic chunk length: the smallest L whose ceil(T / L) chunks fill
// `waves` waves of co-resident threads of the per-step kernels (whole waves:
// no tail).  Fewer waves mean fewer chunk elements for the scan (the DLB
// folds ceil(chunks / resident) per thread), more waves keep the per-step
// kernels closer to the HBM roof; 4 is the measured optimum at T = 2^24
// (profiles/r01_v3: L = 64/74/111/148/222/443 -> 5.08/4.96/4.85/4.99/5.03/
// 5.17 ms per PRTS) ...
// Steps per staged row of the model's smallest dense field (StageMaps::grp):
// chunk starts must fall on row boundaries.
template <typename S, int NX, int NY>
int group_mult(const ModelView<S>& m) {
  const long long st[7] = {m.sf, m.su, m.sq, m.sh, m.sd, m.sr, m.sy};
  const int blk[7] = {NX * NX, NX, NX * NX, NY * NX, NY, NY * NY, NY};
  int g = 1;
  for (int f = 0; f < 7; ++f) {
    const int b = blk[f] * (int)sizeof(S);
    if (b < 16 && 16 % b == 0 && st[f] == blk[f] && 16 / b > g) g = 16 / b;
  }
  return g;
}

template <typename S, int NX, int NY>
long long auto_chunk(long long T, int waves, int mult = 1) {
  const int per_sm = kernel_setup(k_filter_finish<S, NX, NY, true>, kStageNT,
                                  FilterTma<S, NX, NY>::smem_n(FilterTma<S, NX, NY>::finish_stages));
  const long long wave = (long long)device_sms() * (per_sm > 0 ? per_sm : 1) * kStageNT;
  // default: 6 waves (same-box chunk sweep at 2^24, profiles/r02_v4: FP32
  // kernels 2.444 ms at 6 waves, 2.463 at 8, 2.557 at 3; FP64 4.47 at 6 and 8,
  // 4.51-4.53 at 4).  Whole waves matter: 4.5 waves cost FP32 +12 %.
  const int w = waves > 0 ? waves : 6;
  const long long L = (T + wave * w - 1) / (wave * w);
  // ... but at least 64 steps per chunk unless that leaves less than one
  // wave of chunks: short chunks make the per-chunk costs (incoming state,
  // chunk-end element) and the scan's element count dominate
  // (profiles/r01_v7: T = 2^20 with L = 7 / 28: 0.87 / 0.64 ms per PRTS)
  long long Lmin = (T + wave - 1) / wave;
  if (Lmin > 64) Lmin = 64;
  long long r = L < Lmin ? Lmin : (L < 1 ? 1 : L);
  // a multiple of the row grouping of the small dense fields (chunk starts
  // on row boundaries).  (L within +-15 % of this choice measures within run
  // noise, 4.74-4.90 ms at 2^24: profiles/r01_v9/chunk_landscape.txt.)
  if (r > mult) r = (r + mult - 1) / mult * mult;
  return r;
}

// Scratch of one fast run (allocated by fast_prepare).
template <typename S>
struct FastScratch {
  long long nchunks = 0, npad = 0, chunk = 1;
  // component stride of agg / sagg (>= npad) and the slot orders of the
  // filter (forward), smoother (reverse) and PTFS backward (reverse) chunk
  // elements: tile-transposed scan order under the DLB, chunk order else
  long long cap = 0;
  ChunkOrder ford{0, 0, 0}, sord{0, 0, 0}, bord{0, 0, 0};
  ScanPlan plan;
  S *agg = nullptr, *aux1 = nullptr, *aux2 = nullptr;
  S* sagg = nullptr;        // smoother chunk elements (built by the filter finish)
  S* egl = nullptr;         // per-step smoothing elements (PRTS only)
  long long ecap = 0;       // chunk capacity of egl (a multiple of 32: TMA rows)
  bool sagg_valid = false;
  void* dlb = nullptr;
  // sharded PTFS backward finish: the forward half's filtered stats of this
  // shard (dense mean[t][nx], cov[t][nx][nx]) in place of egl
  const S* fmean = nullptr;
  const S* fcov = nullptr;
};

template <typename S, int NX, int NY>
static int fast_prepare_t(const ModelView<S>& m, const FastArgs& a, FastScratch<S>& sc,
                          void* (*alloc)(size_t, void*), void* actx) {
  const long long T = m.t;
  sc.chunk = a.chunk >= 1 ? a.chunk : auto_chunk<S, NX, NY>(T, a.waves, group_mult<S, NX, NY>(m));
  if (a.chunk < 1 && a.alg == 0 && sc.chunk < seq_chunk_floor(T)) {
    const long long mult = group_mult<S, NX, NY>(m);
    sc.chunk = (seq_chunk_floor(T) + mult - 1) / mult * mult;
  }
  sc.nchunks = T > 0 ? (T + sc.chunk - 1) / sc.chunk : 0;
  const bool dlb = a.alg == 6;
  sc.npad = (dlb || a.alg == 0) ? sc.nchunks : (long long)next_pow2(sc.nchunks);
  if (!dlb && sc.npad > 0) {
    sc.plan = make_scan_plan(a.alg, a.sengupta_n, sc.npad);
    if (sc.plan.status) return sc.plan.status;
  }
  constexpr int FS = FLayout<NX>::size;
  const long long a1 = dlb ? 0 : sc.plan.cap1, a2 = dlb ? 0 : sc.plan.cap2;
  const long long nch = sc.nchunks;
  if (dlb && nch > 0) {
    const int pf = dlb_per<FastFilterOps<S, NX>>(nch);
    const int ps = dlb_per<FastSmootherOps<S, NX>>(nch);
    sc.ford = ChunkOrder{nch, pf, 0};
    sc.sord = ChunkOrder{nch, ps, 1};
    sc.bord = ChunkOrder{nch, pf, 1};
    sc.cap = sc.ford.cap() > sc.sord.cap() ? sc.ford.cap() : sc.sord.cap();
  } else {
    sc.ford = sc.sord = sc.bord = ChunkOrder{nch, 0, 0};
    sc.cap = sc.npad;
  }
  sc.agg = (S*)alloc(sizeof(S) * FS * (sc.cap ? sc.cap : 1), actx);
  sc.sagg = (S*)alloc(sizeof(S) * SLayout<NX>::size * (sc.cap ? sc.cap : 1), actx);
  sc.sagg_valid = false;
  sc.egl = nullptr;
  sc.ecap = (sc.nchunks + 31) / 32 * 32;
  if (a.method == 1 || a.method == 2) {
    // PRTS: per-step smoothing elements; PTFS: per-step filtered states
    const int per = a.method == 1 ? EglLayout<NX>::size : StateLayout<NX>::size;
    sc.egl = (S*)alloc(sizeof(S) * (size_t)per * (size_t)sc.chunk *
                           (size_t)(sc.ecap ? sc.ecap : 32),
                       actx);
    if (!sc.egl) return 8;
  }
  sc.aux1 = (S*)alloc(sizeof(S) * FS * (a1 ? a1 : 1), actx);
  sc.aux2 = (S*)alloc(sizeof(S) * FS * (a2 ? a2 : 1), actx);
  sc.dlb = dlb ? alloc(dlb_state_bytes<S, NX>(sc.nchunks), actx) : nullptr;
  if (!sc.agg || !sc.sagg || !sc.aux1 || !sc.aux2 || (dlb && !sc.dlb)) return 8;
  return 0;
}

// phase: 0 filter reduce+scan, 1 filter finish, 2 smoother reduce+scan,
//        3 smoother finish, 4 backward (shifted) reduce+scan, 5 backward
//        finish fused with the two-filter combination.
// `carry` (device, state nx + nx^2) is the boundary state of a sharded run
// (nullptr otherwise); `elem_out` (device, packed element) receives the local
// total of a reduce phase when non-null.
template <typename S, int NX, int NY>
static int fast_phase_t(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a,
                        FastScratch<S>& sc, int phase, S* mean, S* cov, const S* carry,
                        S* elem_out) {
  if (sc.nchunks == 0) return 0;
  const long long Lc = sc.chunk, nch = sc.nchunks, npad = sc.npad;
  FastFilterOps<S, NX> fops{L.err};
  FastSmootherOps<S, NX> sops{L.err};
  auto fill = [&](auto ops, S* buf) {
    if (npad > nch) {
      k_fill_identity<<<blocks_for(npad - nch, kBlock), kBlock, 0, L.stream>>>(
          ops, ElemBuf<S>{buf, npad, npad, 0}, nch, npad);
      L.count("fill_identity");
    }
  };
  const int gs = blocks_for(nch, kStageNT);
  // TMA stages of the per-step inputs (psk_stage.cuh): two for the reduce
  // and backward passes, FilterTma::finish_stages for the filter finish
  const int stage_bytes = FilterTma<S, NX, NY>::smem;
  const int finish_bytes = FilterTma<S, NX, NY>::smem_n(FilterTma<S, NX, NY>::finish_stages);
  const long long nfull = m.t / Lc;  // complete chunks (extent of the tensor maps)
  StageMaps maps;
  if (phase == 0 || phase == 1) {
    const int st = make_stage_maps<S, NX, NY>(m, Lc, nfull, maps);
    if (st) return st;
  }
  switch (phase) {
    case 0:
      kernel_setup(k_filter_reduce<S, NX, NY>, kStageNT, stage_bytes);
      k_filter_reduce<S, NX, NY><<<gs, kStageNT, stage_bytes, L.stream>>>(
          m, maps, Lc, nch, nfull, sc.agg, sc.cap, sc.ford, L.err);
      L.count("filter_reduce");
      fill(fops, sc.agg);
      chunk_scan(L, fops, a, sc.agg, nch, npad, 0, sc.aux1, sc.aux2, sc.plan, sc.dlb, sc.cap);
      if (elem_out) {
        k_extract_elem<<<1, 64, 0, L.stream>>>(sc.agg, sc.cap, sc.ford.at(nch - 1),
                                               FLayout<NX>::size, elem_out);
        L.count("extract_elem");
      }
      break;
    case 1:  // filter finish; for PRTS also folds the smoother chunk elements
      if (a.method == 1) {
        EglStore em;
        const int st = make_egl_store_map<S, NX, NY>(sc.egl, sc.ecap, Lc, em);
        if (st) return st;
        kernel_setup(k_filter_finish<S, NX, NY, true>, kStageNT, finish_bytes);
        k_filter_finish<S, NX, NY, true><<<gs, kStageNT, finish_bytes, L.stream>>>(
            m, maps, Lc, nch, nfull, sc.agg, sc.cap, sc.ford, carry, mean, cov, sc.sagg,
            sc.cap, sc.sord, sc.egl, sc.ecap, L.err, em);
        L.count("filter_finish_smoother_reduce");
      } else {
        EglStore em;
        em.use = 0;
        kernel_setup(k_filter_finish<S, NX, NY, false>, kStageNT, finish_bytes);
        k_filter_finish<S, NX, NY, false><<<gs, kStageNT, finish_bytes, L.stream>>>(
            m, maps, Lc, nch, nfull, sc.agg, sc.cap, sc.ford, carry, mean, cov, nullptr,
            sc.cap, sc.sord, a.method == 2 ? sc.egl : nullptr, sc.ecap, L.err, em);
        L.count("filter_finish");
      }
      sc.sagg_valid = a.method == 1;
      break;
    case 2:
      // the smoother chunk elements and per-step elements come from the
      // PRTS filter finish (phase 1)
      if (!sc.sagg_valid || sc.egl == nullptr) return 7;
      fill(sops, sc.sagg);
      chunk_scan(L, sops, a, sc.sagg, nch, npad, 1, sc.aux1, sc.aux2, sc.plan, sc.dlb, sc.cap);
      if (elem_out) {
        k_extract_elem<<<1, 64, 0, L.stream>>>(sc.sagg, sc.cap, sc.sord.at(0),
                                               SLayout<NX>::size, elem_out);
        L.count("extract_elem");
      }
      break;
    case 3:
    {
      if (sc.egl == nullptr) return 7;
      SmoothMaps sm_maps;
      const int st = make_smooth_maps<S, NX>(sc.egl, sc.ecap, Lc, nfull, mean, cov, sm_maps);
      if (st) return st;
      const int smem = kSmoothNT / 32 * SmoothTma<S, NX>::warp + 1024;
      kernel_setup(k_smoother_finish<S, NX>, kSmoothNT, smem);
      k_smoother_finish<S, NX><<<blocks_for(nch, kSmoothNT), kSmoothNT, smem, L.stream>>>(
          m.t, Lc, nch, nfull, sc.sagg, sc.cap, sc.sord, carry, sm_maps, sc.ecap, mean, cov);
    }
      L.count("smoother_finish");
      sc.sagg_valid = false;
      break;
    case 4: {
      // backward elements: slot i = a(step i+1) -> the filter reduce over the
      // model shifted by one step (chunk c of it = slots [cL, cL + L)), from
      // the identity; chunks past T - 1 steps are pure identity
      const ModelView<S> ms = shift_model(m);
      const long long nch_s = ms.t > 0 ? (ms.t + Lc - 1) / Lc : 0;
      StageMaps smaps;
      const int st = make_stage_maps<S, NX, NY>(ms, Lc, ms.t / Lc, smaps);
      if (st) return st;
      if (nch_s > 0) {
        kernel_setup(k_filter_reduce<S, NX, NY>, kStageNT, stage_bytes);
        k_filter_reduce<S, NX, NY><<<blocks_for(nch_s, kStageNT), kStageNT, stage_bytes,
                                     L.stream>>>(ms, smaps, Lc, nch_s, ms.t / Lc, sc.agg, sc.cap,
                                                 sc.bord, L.err);
        L.count("bwd_reduce");
      }
      if (sc.bord.per > 0) {  // DLB order: the (at most one) identity chunk's slot
        for (long long c = nch_s; c < nch; ++c) {
          const long long q = sc.bord.at(c);
          k_fill_identity<<<1, kBlock, 0, L.stream>>>(fops, ElemBuf<S>{sc.agg, sc.cap, sc.cap, 0},
                                                      q, q + 1);
          L.count("fill_identity");
        }
      } else if (npad > nch_s) {
        k_fill_identity<<<blocks_for(npad - nch_s, kBlock), kBlock, 0, L.stream>>>(
            fops, ElemBuf<S>{sc.agg, npad, npad, 0}, nch_s, npad);
        L.count("fill_identity");
      }
      chunk_scan(L, fops, a, sc.agg, nch, npad, 1, sc.aux1, sc.aux2, sc.plan, sc.dlb, sc.cap);
      if (elem_out) {  // the shard's backward total (reverse scan value of chunk 0)
        k_extract_elem<<<1, 64, 0, L.stream>>>(sc.agg, sc.cap, sc.bord.at(0),
                                               FLayout<NX>::size, elem_out);
        L.count("extract_elem");
      }
      break;
    }
    case 5: {
      const ModelView<S> ms = shift_model(m);
      StageMaps smaps;
      const int st = make_stage_maps<S, NX, NY>(ms, Lc, ms.t / Lc, smaps);
      if (st) return st;
      kernel_setup(k_bwd_finish<S, NX, NY>, kStageNT, stage_bytes);
      k_bwd_finish<S, NX, NY><<<gs, kStageNT, stage_bytes, L.stream>>>(
          ms, smaps, m.t, Lc, nch, ms.t / Lc, sc.agg, sc.cap, sc.bord, sc.egl, sc.ecap, mean,
          cov, carry, sc.fmean, sc.fcov, L.err);
      L.count("bwd_finish_tf_combine");
      break;
    }
    default:
      return 7;
  }
  return 0;
}

template <typename S, int NX, int NY>
static int fast_run_t(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a, S* mean,
                      S* cov, void* (*alloc)(size_t, void*), void* actx) {
  if (m.t == 0) return 0;
  FastScratch<S> sc;
  int st = fast_prepare_t<S, NX, NY>(m, a, sc, alloc, actx);
  if (st) return st;
  const int phases[2][4] = {{0, 1, 2, 3}, {0, 1, 4, 5}};
  const int n = a.method == 0 ? 2 : 4;
  for (int i = 0; i < n; ++i) {
    st = fast_phase_t<S, NX, NY>(L, m, a, sc, phases[a.method == 2][i], mean, cov, nullptr,
                                 nullptr);
    if (st) return st;
  }
  return 0;
}

// PTFS with the forward and the backward pass on two contexts (two GPUs, or
// two streams of one): the backward (shifted-element) reduce + reversed scan
// runs on B concurrently with the forward filter on A; the scanned backward
// chunk elements (nchunks x 56 scalars, not the per-step (eta, J) the
// reference copies, kalman_par.hpp:223-236) are then copied to A, where the
// backward finish fused with the two-filter combination writes the smoothed
// stats.  `mA`/`mB` view the same model on each device.
template <typename S, int NX, int NY>
static int fast_ptfs2_t(ExactLaunch& LA, const ModelView<S>& mA, int devA, ExactLaunch& LB,
                        const ModelView<S>& mB, int devB, FastArgs a, S* mean, S* cov,
                        void* (*allocA)(size_t, void*), void* ctxA,
                        void* (*allocB)(size_t, void*), void* ctxB) {
  if (mA.t == 0) return 0;
  a.method = 2;
  if (a.chunk < 1) {  // same L on both sides
    a.chunk = auto_chunk<S, NX, NY>(mA.t, a.waves, group_mult<S, NX, NY>(mA));
    if (a.alg == 0 && a.chunk < seq_chunk_floor(mA.t)) {
      const long long mult = group_mult<S, NX, NY>(mA);
      a.chunk = (seq_chunk_floor(mA.t) + mult - 1) / mult * mult;
    }
  }
  FastScratch<S> sa, sb;
  cudaSetDevice(devB);
  int st = fast_prepare_t<S, NX, NY>(mB, a, sb, allocB, ctxB);
  if (st) return st;
  st = fast_phase_t<S, NX, NY>(LB, mB, a, sb, 4, nullptr, nullptr, nullptr, nullptr);
  if (st) return st;
  cudaEvent_t done_b;
  if (cudaEventCreateWithFlags(&done_b, cudaEventDisableTiming) != cudaSuccess) return 7;
  // destroyed on every path below (an event still pending in a stream wait is
  // released by the runtime once the wait completes)
  struct EventGuard {
    cudaEvent_t e;
    ~EventGuard() { cudaEventDestroy(e); }
  } guard{done_b};
  cudaEventRecord(done_b, LB.stream);
  cudaSetDevice(devA);
  if (devA != devB) enable_peer(devA, devB);  // NVLink P2P for the element copy
  st = fast_prepare_t<S, NX, NY>(mA, a, sa, allocA, ctxA);
  if (st) return st;
  st = fast_phase_t<S, NX, NY>(LA, mA, a, sa, 0, mean, cov, nullptr, nullptr);
  if (!st) st = fast_phase_t<S, NX, NY>(LA, mA, a, sa, 1, mean, cov, nullptr, nullptr);
  if (st) return st;
  // the forward elements in sa.agg are dead after the forward finish
  cudaStreamWaitEvent(LA.stream, done_b, 0);
  // both sides hold the backward elements in the same slot order
  if (sa.cap != sb.cap || sa.bord.per != sb.bord.per) return 7;
  cudaMemcpyPeerAsync(sa.agg, devA, sb.agg, devB,
                      sizeof(S) * FLayout<NX>::size * (size_t)sa.cap, LA.stream);
  LA.count("ptfs_backward_elements_peer_copy");
  return fast_phase_t<S, NX, NY>(LA, mA, a, sa, 5, mean, cov, nullptr, nullptr);
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
int fast_run(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a, S* mean, S* cov,
             void* (*alloc)(size_t, void*), void* actx) {
#define PSK_CASE(A, B) \
  if (m.nx == A && m.ny == B) return fast_run_t<S, A, B>(L, m, a, mean, cov, alloc, actx);
  PSK_FAST_DIMS(PSK_CASE)
#undef PSK_CASE
  return -1;
}

template <typename S>
int fast_ptfs2(ExactLaunch& LA, const ModelView<S>& mA, int devA, ExactLaunch& LB,
               const ModelView<S>& mB, int devB, const FastArgs& a, S* mean, S* cov,
               void* (*allocA)(size_t, void*), void* ctxA, void* (*allocB)(size_t, void*),
               void* ctxB) {
#define PSK_CASE(A, B)                                                                      \
  if (mA.nx == A && mA.ny == B)                                                             \
    return fast_ptfs2_t<S, A, B>(LA, mA, devA, LB, mB, devB, a, mean, cov, allocA, ctxA, \
                                 allocB, ctxB);
  PSK_FAST_DIMS(PSK_CASE)
#undef PSK_CASE
  return -1;
}

// one phase of a sharded run; `scratch` is an opaque FastScratch<S> owned by
// the caller (allocated on phase 0 / 2 with the persistent allocator)
// phase 5 (sharded PTFS backward finish) reads the forward states from the
// dense (fmean, fcov) arrays instead of the scratch the forward finish fills.
template <typename S>
int fast_shard_phase(ExactLaunch& L, const ModelView<S>& m, const FastArgs& a, int phase,
                     void** scratch, S* mean, S* cov, const S* carry, S* elem_out,
                     void* (*alloc)(size_t, void*), void* actx, const S* fmean,
                     const S* fcov) {
  auto* sc = static_cast<FastScratch<S>*>(*scratch);
  if (!sc) {
    sc = new FastScratch<S>();
    *scratch = sc;
  }
  sc->fmean = fmean;
  sc->fcov = fcov;
#define PSK_CASE(A, B)                                                           \
  if (m.nx == A && m.ny == B) {                                                  \
    if (phase == 0 || phase == 4) {                                              \
      int st = fast_prepare_t<S, A, B>(m, a, *sc, alloc, actx);                    \
      if (st) return st;                                                         \
    }                                                                            \
    return fast_phase_t<S, A, B>(L, m, a, *sc, phase, mean, cov, carry, elem_out); \
  }
  PSK_FAST_DIMS(PSK_CASE)
#undef PSK_CASE
  return -1;
}
template <typename S>
void fast_shard_release(void* scratch) {
  delete static_cast<FastScratch<S>*>(scratch);
}

// folds of gathered shard elements (one thread; count <= number of ranks)
template <typename S>
int fast_fold(ExactLaunch& L, int kind, int nx, const S* aggs, int count, S* out) {
  if (count <= 0) return 7;
#define PSK_FOLD(N)                                                            \
  if (nx == N) {                                                               \
    if (kind == 0)                                                             \
      k_fold_filter<S, N><<<1, 32, 0, L.stream>>>(aggs, count, out, L.err);    \
    else if (kind == 1)                                                        \
      k_fold_smoother<S, N><<<1, 32, 0, L.stream>>>(aggs, count, out);         \
    else                                                                       \
      k_fold_backward<S, N><<<1, 32, 0, L.stream>>>(aggs, count, out, L.err);  \
    L.count(kind == 0 ? "fold_filter" : kind == 1 ? "fold_smoother" : "fold_backward"); \
    return 0;                                                                  \
  }
  PSK_FOLD(1) PSK_FOLD(2) PSK_FOLD(3) PSK_FOLD(4)
#undef PSK_FOLD
  return -1;
}

}  // namespace psk
