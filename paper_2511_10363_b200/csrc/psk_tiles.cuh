// psk_tiles.cuh -- shared-memory block execution of the intra-tile levels of
// the reference's tree scans (fast mode).
//
// In the up-sweep (scan.hpp:261-279) and in the Blelloch / Ladner-Fischer
// down-sweeps (scan.hpp:281-367) every level whose block width d2 is at most
// kTile combines elements that lie in the same kTile-aligned tile (the
// Ladner-Fischer down-sweep reads, besides, the previous tile's last element,
// which is final once the wider levels are done and which no intra-tile level
// writes).  Those levels -- log2(kTile) of them at each end of the sweep --
// run here in ONE kernel per end: a CTA loads its tile into shared memory,
// performs the levels with the reference's index maps separated by block
// barriers, and writes the tile back.  The wider levels touch only the tiles'
// last elements, so the sweep recurses on the view of those roots; the
// innermost view (<= kTile elements) does its whole sweep in one CTA.  A sweep
// over n elements is 2 ceil(log_kTile n) - 1 launches instead of ~2 log2 n.
// Every combine happens with the same operands in the same order as the
// level-by-level execution, so the result is identical.  (Hillis-Steele levels read
// across tiles and the Sengupta hybrid keeps its arena: both stay level-by-
// level.)  Blelloch's copy of the originals and its final combine with them
// (scan.hpp:290, 333-340) are fused into the two kernels.
#pragma once
#include <cuda_runtime.h>

#include "psk_common.cuh"

namespace psk {

constexpr int kTile = 128;
constexpr int kTileSlots = kTile + 1;  // + the previous tile's last element

template <class Ops>
__device__ __forceinline__ void tile_swap(const ElemBuf<typename Ops::S>& sb, int j, int k) {
  using S = typename Ops::S;
  for (int c = 0; c < Ops::kSize; ++c) {  // the thread's own pair of slots
    S* pj = sb.p + (size_t)c * sb.cap + j;
    S* pk = sb.p + (size_t)c * sb.cap + k;
    const S x = *pj;
    *pj = *pk;
    *pk = x;
  }
}
template <class Ops>
__device__ __forceinline__ void tile_comb(const Ops& ops, int rev,
                                          const ElemBuf<typename Ops::S>& sb, int d, int l,
                                          int r) {
  if (!rev)
    ops.combine(sb, d, sb, l, sb, r);
  else
    ops.combine(sb, d, sb, r, sb, l);
}

// A strided view of the logical buffer: view element i is element
// off + i * stride.  Every level of the up- and down-sweeps wider than a tile
// touches only the tiles' last elements (indices = -1 mod the tile width), so
// the sweep recurses on the view of those roots (stride x kTile).
struct TileView {
  long long n, stride, off;
  __device__ __forceinline__ long long at(long long i) const { return off + i * stride; }
};

// up-sweep levels d = 0 .. log2(tile) - 1 on every tile of the view; `orig`
// (Blelloch, outermost view only) receives a copy of the inputs
// Sengupta's reduce passes (scan.hpp:390-410) written by the tile up-sweep:
// the up-sweep node at tile position t 2^d + 2^d - 1 IS the level-d arena
// node (tile q) * (kTile >> d) + t; `off[d]` = arena offset of level d.
struct ArenaOut {
  long long off[8];
};

template <class Ops>
__global__ void __launch_bounds__(kTile)
    k_tile_up(Ops ops, ElemBuf<typename Ops::S> a, ElemBuf<typename Ops::S> orig, TileView v,
              ElemBuf<typename Ops::S> arena, ArenaOut ao) {
  using S = typename Ops::S;
  extern __shared__ __align__(16) unsigned char tile_smem[];
  const ElemBuf<S> sb{reinterpret_cast<S*>(tile_smem), kTileSlots, kTileSlots, 0};
  const long long base = (long long)blockIdx.x * kTile;
  const int t = threadIdx.x;
  const long long g = a.phys(v.at(base + t));
  ops.assign(sb, t, a, g);
  if (orig.p != nullptr) ops.assign(orig, orig.phys(v.at(base + t)), a, g);
  __syncthreads();
  int lev = 0;
#pragma unroll 1
  for (int d1 = 1; d1 < kTile; d1 <<= 1) {
    const int d2 = d1 << 1;
    ++lev;
    if (t < kTile / d2) {
      tile_comb(ops, a.rev, sb, t * d2 + d2 - 1, t * d2 + d1 - 1, t * d2 + d2 - 1);
      if (arena.p != nullptr)
        ops.assign(arena, arena.phys(ao.off[lev] + (long long)blockIdx.x * (kTile / d2) + t), sb,
                   t * d2 + d2 - 1);
    }
    __syncthreads();
  }
  ops.assign(a, g, sb, t);
}

// Down-sweep levels d = log2(tile) - 1 .. 0 on every tile of the view:
// Ladner-Fischer (BLELLOCH = false, scan.hpp:343-367; the pair of width 2^d
// whose left end is the previous tile's last element reads it from global
// memory: it is final, no intra-tile level writes it) or Blelloch
// (scan.hpp:320-331), then for Blelloch's outermost view a_i (x) orig_i
// (scan.hpp:333-340).
// With `arena` given (Sengupta, BLELLOCH = false): the distribute passes
// d = log2(tile) - 1 .. 0 (scan.hpp:413-443) in place are exactly these
// Ladner-Fischer pairs, once the tile roots hold their final prefixes --
// the arena's level-log2(tile) nodes after the wider distribute passes.
template <class Ops, bool BLELLOCH>
__global__ void __launch_bounds__(kTile)
    k_tile_down(Ops ops, ElemBuf<typename Ops::S> a, ElemBuf<typename Ops::S> orig, TileView v,
                ElemBuf<typename Ops::S> arena, long long root_off) {
  using S = typename Ops::S;
  extern __shared__ __align__(16) unsigned char tile_smem[];
  const ElemBuf<S> sb{reinterpret_cast<S*>(tile_smem), kTileSlots, kTileSlots, 0};
  const long long base = (long long)blockIdx.x * kTile;
  const int t = threadIdx.x;
  constexpr int kHalo = kTile;
  const long long g = a.phys(v.at(base + t));
  ops.assign(sb, t, a, g);
  if (!BLELLOCH && t == 0 && base > 0) ops.assign(sb, kHalo, a, a.phys(v.at(base - 1)));
  if (arena.p != nullptr) {
    __syncthreads();
    if (t == kTile - 1) ops.assign(sb, t, arena, arena.phys(root_off + blockIdx.x));
    if (t == 0 && base > 0) ops.assign(sb, kHalo, arena, arena.phys(root_off + blockIdx.x - 1));
  }
  __syncthreads();
#pragma unroll 1
  for (int d1 = kTile / 2; d1 >= 1; d1 >>= 1) {
    const int d2 = d1 << 1;
    if (BLELLOCH) {
      // t' = a_j; a_j = a_k; a_k = a_k (x) t'  ==  a_j <- a_k (x) a_j, swap
      if (t < kTile / d2) {
        const int j = t * d2 + d1 - 1, k = t * d2 + d2 - 1;
        tile_comb(ops, a.rev, sb, j, k, j);
        tile_swap<Ops>(sb, j, k);
      }
    } else if (t < kTile / d2 && (t > 0 || base > 0)) {
      // pairs (q d2 - 1, q d2 - 1 + d1); q = 0: the previous tile's last
      const int i = t == 0 ? kHalo : t * d2 - 1;
      tile_comb(ops, a.rev, sb, t * d2 + d1 - 1, i, t * d2 + d1 - 1);
    }
    __syncthreads();
  }
  if (BLELLOCH && orig.p != nullptr) {
    if (!a.rev)
      ops.combine(sb, t, sb, t, orig, orig.phys(v.at(base + t)));
    else
      ops.combine(sb, t, orig, orig.phys(v.at(base + t)), sb, t);
  }
  ops.assign(a, g, sb, t);
}

// A whole sweep of a view of n <= kTile elements in one CTA: the up-sweep,
// Blelloch's identity at the last element (scan.hpp:318), the down-sweep and,
// for Blelloch's outermost view, the final combine with the originals.
template <class Ops, bool BLELLOCH>
__global__ void __launch_bounds__(kTile)
    k_tile_all(Ops ops, ElemBuf<typename Ops::S> a, ElemBuf<typename Ops::S> orig, TileView v,
               ElemBuf<typename Ops::S> copy_to) {
  using S = typename Ops::S;
  extern __shared__ __align__(16) unsigned char tile_smem[];
  const ElemBuf<S> sb{reinterpret_cast<S*>(tile_smem), kTileSlots, kTileSlots, 0};
  const int n = (int)v.n;
  const int t = threadIdx.x;
  const long long g = t < n ? a.phys(v.at(t)) : 0;
  if (t < n) {
    ops.assign(sb, t, a, g);
    if (copy_to.p != nullptr) ops.assign(copy_to, copy_to.phys(v.at(t)), a, g);
  }
  __syncthreads();
#pragma unroll 1
  for (int d1 = 1; d1 < n; d1 <<= 1) {
    const int d2 = d1 << 1;
    if (t < n / d2) tile_comb(ops, a.rev, sb, t * d2 + d2 - 1, t * d2 + d1 - 1, t * d2 + d2 - 1);
    __syncthreads();
  }
  if (BLELLOCH && t == 0) ops.identity(sb, n - 1);
  __syncthreads();
#pragma unroll 1
  for (int d1 = n / 2; d1 >= 1; d1 >>= 1) {
    const int d2 = d1 << 1;
    if (BLELLOCH) {
      if (t < n / d2) {
        const int j = t * d2 + d1 - 1, k = t * d2 + d2 - 1;
        tile_comb(ops, a.rev, sb, j, k, j);
        tile_swap<Ops>(sb, j, k);
      }
    } else if (t > 0 && t < n / d2) {  // Ladner-Fischer: blocks - 1 pairs
      tile_comb(ops, a.rev, sb, t * d2 + d1 - 1, t * d2 - 1, t * d2 + d1 - 1);
    }
    __syncthreads();
  }
  if (t < n) {
    if (BLELLOCH && orig.p != nullptr) {
      if (!a.rev)
        ops.combine(sb, t, sb, t, orig, orig.phys(v.at(t)));
      else
        ops.combine(sb, t, orig, orig.phys(v.at(t)), sb, t);
    }
    ops.assign(a, g, sb, t);
  }
}

}  // namespace psk
