// psk_dlb.cuh -- single-pass decoupled look-back scan (NEW: not in the
// reference; appended as ScanAlg value 6 after SenguptaB, scan.hpp:32-39).
//
// One CTA of kDlbThreads threads scans a tile of kDlbThreads * K consecutive
// elements (K per thread, chosen on the host so that all tiles of a typical
// chunk scan are resident in one wave):
//   1. tile ticket from a global counter (forward progress: every tile with a
//      smaller ticket is running or done);
//   2. each thread folds its K consecutive elements serially (work-efficient);
//   3. the 128 thread aggregates are scanned in shared memory (up-sweep +
//      Ladner-Fischer down-sweep, the index maps of scan.hpp:261-279 and
//      343-367 applied to the tile); the thread-inclusive prefixes are parked
//      in global scratch;
//   4. the tile aggregate is published (flag A; tile 0 publishes its inclusive
//      prefix, flag P, directly);
//   5. look-back, CTA-parallel: the flags of 128-wide windows of
//      predecessors are inspected until the nearest P (inclusive prefix) is
//      found; the P and the aggregates after it are then split into 128
//      contiguous blocks, each thread folds its block in time order and a
//      7-level ordered tree in shared memory reduces the blocks
//      (non-commutative) -- the exclusive prefix of the tile;
//   6. the inclusive prefix of the tile is published (flag P) and every thread
//      re-folds its K elements from (exclusive tile prefix (x) thread
//      exclusive prefix), writing the inclusive prefixes in place.
// The element payload (56 scalars at nx=4) is far wider than an atomic, so it
// is published as payload + release flag and read with L1-bypassing loads
// after an acquire load of the flag.  Reverse scans use the Reversed<E> index
// map with flipped operands (scan.hpp:149-177).
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "psk_common.cuh"
#include "psk_exact.h"

namespace psk {

constexpr int kDlbThreads = 128;
static_assert(kDlbThreads == kOrderNT, "ChunkOrder tiles are look-back tiles");
constexpr int kDlbLevels = 7;  // log2(kDlbThreads)
static_assert((1 << kDlbLevels) == kDlbThreads, "CTA must be 2^kDlbLevels threads");
constexpr int kDlbSlots = kDlbThreads + 2;  // + exclusive tile prefix + scratch

// Optional phase trace (tools/dlb_trace.py): thread 0 of every tile stamps
// %globaltimer at the phase boundaries into trace[tile * 8 + i].
__device__ __forceinline__ void dlb_stamp(unsigned long long* trace, long long tile, int i) {
  if (trace != nullptr && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    trace[tile * 8 + i] = g;
  }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Elements per thread: the smallest K >= 1 that keeps every tile resident in
// ONE wave (`resident` = co-resident CTAs of k_dlb on the device, from the
// occupancy calculator), so the look-back never waits on a tile that has not
// started and spans at most ceil(resident / 128) windows.
inline int dlb_per_thread(long long n, long long resident) {
  const long long target = (resident > 0 ? resident : 148) * kDlbThreads;
  long long k = (n + target - 1) / target;
  if (k < 1) k = 1;
  if (k > 64) k = 64;
  return (int)k;
}
inline long long dlb_tiles(long long n, int per) {
  const long long tile = (long long)kDlbThreads * per;
  return (n + tile - 1) / tile;
}
__host__ __device__ inline size_t dlb_head_bytes(long long ntiles) {
  return 256 + ((size_t)ntiles * 4 + 255) / 256 * 256;
}
// Published tile payloads are AoS, one element per kDlbStride scalars (whole
// 128-byte lines for FP64): a cache line never mixes tiles, so no line can
// be cached by a reader before its tile's flag is set.
constexpr int kDlbStride = 64;
// state layout: [ticket u32 | pad][flags u32 x ntiles][agg x ntiles (AoS)]
//               [incl x ntiles (AoS)][thread prefixes FS x ntiles*kDlbThreads]
// sized for the worst case K = 1 (one element per thread)
template <typename S, int NX>
inline size_t dlb_state_bytes(long long n) {
  const long long nt = dlb_tiles(n, 1);
  const size_t fs = (size_t)(3 * NX * NX + 2 * NX);
  return dlb_head_bytes(nt) + sizeof(S) * (size_t)nt * (2 * kDlbStride + fs * kDlbThreads);
}

// The warp-shuffle tile scan needs two elements in registers per thread:
// used where they fit (FP32 elements, the 36-scalar FP64 smoothing element);
// the 56-double filtering element keeps the shared-memory sweeps.
template <class Ops>
constexpr bool dlb_shuffle() {
  return Ops::kSize * sizeof(typename Ops::S) <= 320;
}

template <class Ops>
__global__ void __launch_bounds__(kDlbThreads)
    k_dlb(Ops ops, typename Ops::S* buf, long long n, long long cap, int rev, int perm,
          char* state, long long ntiles, int per, unsigned long long* trace) {
  using S = typename Ops::S;
  extern __shared__ __align__(16) unsigned char dlb_smem[];
  S* sm = reinterpret_cast<S*>(dlb_smem);
  const ElemBuf<S> sb{sm, kDlbSlots, kDlbSlots, 0};
  const ElemBuf<S> gb{buf, cap, n, 0};
  unsigned* ticket = reinterpret_cast<unsigned*>(state);
  unsigned* flags = reinterpret_cast<unsigned*>(state + 256);
  static_assert(Ops::kSize <= kDlbStride, "element wider than the payload stride");
  S* pagg = reinterpret_cast<S*>(state + dlb_head_bytes(ntiles));
  S* pincl = pagg + (size_t)kDlbStride * ntiles;
  S* pthr = pincl + (size_t)kDlbStride * ntiles;
  const long long thr_cap = ntiles * kDlbThreads;
  // AoS views: element p at index p * kDlbStride (component stride 1)
  const ElemBuf<S> ab{pagg, 1, ntiles * kDlbStride, 0};
  const ElemBuf<S> ib{pincl, 1, ntiles * kDlbStride, 0};
  const ElemBuf<S> tb{pthr, thr_cap, thr_cap, 0};
  constexpr int kExcl = kDlbThreads, kTmp = kDlbThreads + 1;
  __shared__ unsigned s_tile;
  __shared__ int s_stop;
  const int t = threadIdx.x;
  if (t == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const long long tile = s_tile;
  dlb_stamp(trace, tile, 0);
  // logical (x) on (buffer, index) pairs: reversed scans flip the operands
  // (selected, not branched: one inlined combine per call site)
  auto lcomb = [&](const ElemBuf<S>& d, long long di, const ElemBuf<S>& l, long long li,
                   const ElemBuf<S>& r, long long ri) {
    ops.combine(d, di, rev ? r : l, rev ? ri : li, rev ? l : r, rev ? li : ri);
  };
  // slot of scan element g: the ChunkOrder of the buffer (perm: the tile
  // transpose, already in scan order) or the reference's Reversed map
  const ChunkOrder ord{n, per, 0};
  auto phys = [&](long long g) { return perm ? ord.at(g) : (rev ? n - 1 - g : g); };

  // 2. serial fold of this thread's K consecutive elements into slot t
  const long long g0 = (tile * kDlbThreads + t) * per;
  const long long g1 = g0 + per < n ? g0 + per : n;
  if (g0 < n) {
    ops.assign(sb, t, gb, phys(g0));
    for (long long g = g0 + 1; g < g1; ++g) lcomb(sb, t, sb, t, gb, phys(g));
  } else {
    ops.identity(sb, t);
  }
  __syncthreads();
  dlb_stamp(trace, tile, 1);
  // 3. tile scan of the thread aggregates
  if constexpr (dlb_shuffle<Ops>()) {
    // warp-shuffle scans: Hillis-Steele (Kogge-Stone) over the 32 lanes of
    // each warp with the elements in registers (scan.hpp:214-259's index map
    // at warp scope, 5 levels, no barriers), then every warp applies the
    // ordered fold of the earlier warps' totals from shared memory
    const int lane = t & 31, w = t >> 5;
    auto x = ops.get(sb, t);
#pragma unroll 1
    for (int d = 1; d < 32; d <<= 1) {
      const auto y = Ops::shfl(x, [&](S v) { return __shfl_up_sync(0xffffffffu, v, d); });
      if (lane >= d) x = rev ? ops.comb(x, y) : ops.comb(y, x);
    }
    ops.put(sb, t, x);
    __syncthreads();
    if (w > 0) {
      auto p = ops.get(sb, 31);
#pragma unroll 1
      for (int v = 1; v < w; ++v) {
        const auto q = ops.get(sb, 32 * v + 31);
        p = rev ? ops.comb(q, p) : ops.comb(p, q);
      }
      x = rev ? ops.comb(x, p) : ops.comb(p, x);
    }
    __syncthreads();
    if (w > 0) ops.put(sb, t, x);
    __syncthreads();
  } else {
    // up-sweep, then Ladner-Fischer down-sweep in shared memory
#pragma unroll 1
    for (int d = 0; d < kDlbLevels; ++d) {
      const int d1 = 1 << d, d2 = d1 << 1;
      if (t < kDlbThreads / d2) {
        const int j = t * d2 + d1 - 1, k = t * d2 + d2 - 1;
        lcomb(sb, k, sb, j, sb, k);
      }
      __syncthreads();
    }
#pragma unroll 1
    for (int d = kDlbLevels - 1; d >= 0; --d) {
      const int d1 = 1 << d, d2 = d1 << 1, blocks = kDlbThreads / d2;
      if (blocks > 1 && t < blocks - 1) {
        const int i = (t + 1) * d2 - 1, j = i + d1;
        lcomb(sb, j, sb, i, sb, j);
      }
      __syncthreads();
    }
  }
  dlb_stamp(trace, tile, 2);
  // 4. publish the tile aggregate (tile 0: its inclusive prefix); park the
  // thread-inclusive prefixes in global scratch (the slots become the window)
  constexpr int last = kDlbThreads - 1;
  if (tile > 0) ops.assign(tb, tile * kDlbThreads + t, sb, t);
  if (t == 0) {
    ops.assign(tile == 0 ? ib : ab, tile * kDlbStride, sb, last);
    __threadfence();
    st_release(flags + tile, tile == 0 ? 2u : 1u);
    if (tile > 0) ops.assign(sb, kTmp, sb, last);  // keep the tile aggregate
  }
  // tile 0: the tile prefix is the identity; slot t already holds the
  // thread-inclusive prefix (shifted to thread-exclusive below)
  if (tile > 0) {
    // 5a. look-back for the nearest predecessor with an inclusive prefix
    // (flag P), over windows of kDlbThreads flags -- no combines yet; every
    // predecessor after it has published its aggregate (flag A) by then
    long long lo = 0;
    long long base = tile - 1;
#pragma unroll 1
    while (true) {
      if (t == 0) s_stop = kDlbThreads;
      __syncthreads();
      const long long pt = base - t;
      if (pt >= 0) {
        unsigned f;
        while ((f = ld_acquire(flags + pt)) == 0u) {
        }
        if (f == 2u) atomicMin(&s_stop, t);
      }
      __syncthreads();
      const int stop = s_stop;  // nearest P (kDlbThreads: none in the window)
      if (stop < kDlbThreads) {
        lo = base - stop;
        break;
      }
      base -= kDlbThreads;  // tile 0 always carries P: the loop ends
    }
    // 5b. the exclusive prefix = incl(lo) (x) agg(lo+1) (x) ... (x) agg(tile-1):
    // thread t folds the contiguous block [lo + t k, lo + (t+1) k) in time
    // order into slot t, then an ordered 7-level tree over the slots -- k - 1
    // + 7 combine latencies for any distance (a window-by-window reduction
    // costs 7 per 128 predecessors)
    {
      const long long m = tile - lo;
      const long long kb = (m + kDlbThreads - 1) / kDlbThreads;
      const long long b0 = lo + t * kb;
      const long long b1 = b0 + kb < tile ? b0 + kb : tile;
      if (b0 < b1) {
        ops.assign(sb, t, b0 == lo ? ib : ab, b0 * kDlbStride);
        for (long long p = b0 + 1; p < b1; ++p) lcomb(sb, t, sb, t, ab, p * kDlbStride);
      } else {
        ops.identity(sb, t);
      }
      __syncthreads();
#pragma unroll 1
      for (int d = 0; d < kDlbLevels; ++d) {
        const int s = 1 << d;
        if ((t & (2 * s - 1)) == 0) lcomb(sb, t, sb, t, sb, t + s);
        __syncthreads();
      }
      if (t == 0) ops.assign(sb, kExcl, sb, 0);
      __syncthreads();
    }
    dlb_stamp(trace, tile, 3);
    // 6. publish the inclusive prefix of the tile
    if (t == 0) {
      lcomb(sb, kTmp, sb, kExcl, sb, kTmp);
      ops.assign(ib, tile * kDlbStride, sb, kTmp);
      __threadfence();
      st_release(flags + tile, 2u);
    }
    __syncthreads();
  }
  dlb_stamp(trace, tile, 4);
  // thread-exclusive prefix: (tile exclusive) (x) (thread-inclusive of t-1)
  if (tile == 0) {
    // shift slot t-1 -> t through registers (all reads before all writes)
    S v[Ops::kSize];
    if (t > 0) {
#pragma unroll
      for (int c = 0; c < Ops::kSize; ++c) v[c] = sm[c * kDlbSlots + t - 1];
    }
    __syncthreads();
    if (t > 0) {
#pragma unroll
      for (int c = 0; c < Ops::kSize; ++c) sm[c * kDlbSlots + t] = v[c];
    }
    __syncthreads();
    if (g0 < n) {
      long long g = g0;
      if (t == 0) {  // no prefix: the first element is its own prefix
        ++g;
        ops.assign(sb, t, gb, phys(g0));
      }
      for (; g < g1; ++g) {
        lcomb(sb, t, sb, t, gb, phys(g));
        ops.assign(gb, phys(g), sb, t);
      }
    }
  } else {
    if (g0 < n) {
      if (t == 0)
        ops.assign(sb, t, sb, kExcl);
      else
        lcomb(sb, t, sb, kExcl, tb, tile * kDlbThreads + t - 1);
      for (long long g = g0; g < g1; ++g) {
        lcomb(sb, t, sb, t, gb, phys(g));
        ops.assign(gb, phys(g), sb, t);
      }
    }
  }
  __syncthreads();
  dlb_stamp(trace, tile, 5);
}

// Elements per thread of a k_dlb<Ops> scan of n elements on this device
// (also the `per` of the ChunkOrder its buffer is stored in).
template <class Ops>
int dlb_per(long long n) {
  using S = typename Ops::S;
  const size_t smem = sizeof(S) * (size_t)Ops::kSize * kDlbSlots;
  const int per_sm = kernel_setup(k_dlb<Ops>, kDlbThreads, (int)smem);
  return dlb_per_thread(n, (long long)device_sms() * per_sm);
}

// `cap`: component stride of buf; `perm`: buf is stored in ChunkOrder{n,
// dlb_per<Ops>(n), rev} (scan-order slots, tile-transposed), else in chunk
// order read through the Reversed map when rev.
template <class Ops>
void dlb_scan(ExactLaunch& L, const Ops& ops, typename Ops::S* buf, long long n,
              long long cap, int rev, int perm, void* state) {
  using S = typename Ops::S;
  if (n <= 0) return;
  const size_t smem = sizeof(S) * (size_t)Ops::kSize * kDlbSlots;
  const int per = dlb_per<Ops>(n);
  const long long ntiles = dlb_tiles(n, per);
  cudaMemsetAsync(state, 0, dlb_head_bytes(ntiles), L.stream);
  unsigned long long* trace = ntiles <= L.dlb_trace_cap ? L.dlb_trace : nullptr;
  k_dlb<Ops><<<(unsigned)ntiles, kDlbThreads, smem, L.stream>>>(
      ops, buf, n, cap, rev, perm, reinterpret_cast<char*>(state), ntiles, per, trace);
  if (trace != nullptr) {  // diagnostics only: synchronises the stream
    std::vector<unsigned long long> h((size_t)ntiles * 8);
    cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, L.stream);
    cudaStreamSynchronize(L.stream);
    FILE* f = std::fopen(L.dlb_trace_path.c_str(), "ab");
    if (f) {
      const long long hdr[4] = {ntiles, per, (long long)Ops::kSize, n};
      std::fwrite(hdr, sizeof(hdr), 1, f);
      std::fwrite(h.data(), 8, h.size(), f);
      std::fclose(f);
    }
  }
  L.count("chunk_scan_dlb");
}

}  // namespace psk
