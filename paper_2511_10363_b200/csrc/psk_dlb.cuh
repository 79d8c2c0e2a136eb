// psk_dlb.cuh -- single-pass decoupled look-back scan (NEW: not in the
// reference; appended as ScanAlg value 6 after SenguptaB, scan.hpp:32-39).
//
// Each CTA takes the next tile of TILE elements from a global ticket counter
// (forward progress: every predecessor tile is running or done), scans it in
// shared memory with a work-efficient up-sweep / Ladner-Fischer down-sweep
// (the pattern of scan.hpp:261-279 and 343-367 applied to the tile),
// publishes its aggregate (flag A) immediately, looks back over the
// predecessors' published aggregates / inclusive prefixes (non-commutative:
// predecessors are folded on the LEFT), publishes its inclusive prefix (flag
// P) and applies the exclusive prefix to its elements.  The element payload
// (56 scalars at nx=4) is far wider than an atomic, so it is published as
// payload + release flag and read back with L1-bypassing loads after an
// acquire load of the flag.  Reverse scans use the Reversed<E> index map with
// flipped operands (scan.hpp:149-177).
#pragma once
#include <cuda_runtime.h>

#include "psk_common.cuh"
#include "psk_exact.h"

namespace psk {

constexpr int kDlbTile = 128;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// state layout: [ticket u32 | pad][flags u32 x ntiles][agg S x size x ntiles]
//               [incl S x size x ntiles]
template <typename S, int NX>
inline size_t dlb_state_bytes(long long n) {
  const long long nt = (n + kDlbTile - 1) / kDlbTile;
  const size_t head = 256 + ((size_t)nt * 4 + 255) / 256 * 256;
  return head + 2 * sizeof(S) * (size_t)(3 * NX * NX + 2 * NX) * (size_t)nt;
}

template <class Ops>
__global__ void __launch_bounds__(kDlbTile)
    k_dlb(Ops ops, typename Ops::S* buf, long long n, int rev, char* state,
          long long ntiles) {
  using S = typename Ops::S;
  constexpr int FS = Ops::kSize;
  extern __shared__ __align__(16) unsigned char dlb_smem[];
  S* sm = reinterpret_cast<S*>(dlb_smem);
  const int cap = kDlbTile + 2;  // slot kDlbTile = exclusive prefix, +1 scratch
  const ElemBuf<S> sb{sm, cap, cap, 0};
  const ElemBuf<S> gb{buf, n, n, 0};
  unsigned* ticket = reinterpret_cast<unsigned*>(state);
  unsigned* flags = reinterpret_cast<unsigned*>(state + 256);
  const size_t head = 256 + ((size_t)ntiles * 4 + 255) / 256 * 256;
  S* pagg = reinterpret_cast<S*>(state + head);
  S* pincl = pagg + (size_t)FS * ntiles;
  __shared__ unsigned s_tile;
  const int t = threadIdx.x;
  if (t == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const long long tile = s_tile;
  const long long g = tile * kDlbTile + t;  // logical index
  // logical (x) on the shared tile: reversed scans flip the operands
  auto lcomb = [&](int dst, int l, int r) {
    if (!rev)
      ops.combine(sb, dst, sb, l, sb, r);
    else
      ops.combine(sb, dst, sb, r, sb, l);
  };
  if (g < n) {
    const long long p = rev ? n - 1 - g : g;
    ops.assign(sb, t, gb, p);
  } else {
    ops.identity(sb, t);
  }
  __syncthreads();
  // tile scan: up-sweep then Ladner-Fischer down-sweep
  constexpr int kLevels = 7;  // log2(kDlbTile)
  static_assert((1 << kLevels) == kDlbTile, "tile must be 2^kLevels");
#pragma unroll 1
  for (int d = 0; d < kLevels; ++d) {
    const int d1 = 1 << d, d2 = d1 << 1;
    if (t < kDlbTile / d2) {
      const int j = t * d2 + d1 - 1, k = t * d2 + d2 - 1;
      lcomb(k, j, k);
    }
    __syncthreads();
  }
#pragma unroll 1
  for (int d = kLevels - 1; d >= 0; --d) {
    const int d1 = 1 << d, d2 = d1 << 1, blocks = kDlbTile / d2;
    if (blocks > 1 && t < blocks - 1) {
      const int i = (t + 1) * d2 - 1, j = i + d1;
      lcomb(j, i, j);
    }
    __syncthreads();
  }
  // publish + look-back (one thread; the payload is FS scalars)
  const ElemBuf<S> ab{pagg, ntiles, ntiles, 0};
  const ElemBuf<S> ib{pincl, ntiles, ntiles, 0};
  if (t == 0) {
    const int last = kDlbTile - 1;
    if (tile == 0) {
      ops.assign(ib, tile, sb, last);
      __threadfence();
      st_release(flags + tile, 2u);
    } else {
      ops.assign(ab, tile, sb, last);
      __threadfence();
      st_release(flags + tile, 1u);
      bool have = false;
      for (long long pt = tile - 1; pt >= 0; --pt) {
        unsigned f;
        while ((f = ld_acquire(flags + pt)) == 0u) {
        }
        const S* src = f == 2u ? pincl : pagg;
        for (int c = 0; c < FS; ++c)
          sm[c * cap + kDlbTile + 1] = __ldcg(src + (size_t)c * ntiles + pt);
        if (!have) {
          ops.assign(sb, kDlbTile, sb, kDlbTile + 1);
          have = true;
        } else {
          lcomb(kDlbTile, kDlbTile + 1, kDlbTile);  // X_pt (x) excl
        }
        if (f == 2u) break;
      }
      lcomb(kDlbTile + 1, kDlbTile, last);  // inclusive = excl (x) aggregate
      ops.assign(ib, tile, sb, kDlbTile + 1);
      __threadfence();
      st_release(flags + tile, 2u);
    }
  }
  __syncthreads();
  if (tile > 0) lcomb(t, kDlbTile, t);
  if (g < n) {
    const long long p = rev ? n - 1 - g : g;
    ops.assign(gb, p, sb, t);
  }
}

template <class Ops>
void dlb_scan(ExactLaunch& L, const Ops& ops, typename Ops::S* buf,
              long long n, int rev, typename Ops::S* /*unused*/, void* state) {
  using S = typename Ops::S;
  if (n <= 0) return;
  const long long ntiles = (n + kDlbTile - 1) / kDlbTile;
  const size_t head = 256 + ((size_t)ntiles * 4 + 255) / 256 * 256;
  cudaMemsetAsync(state, 0, head, L.stream);
  const size_t smem = sizeof(S) * (size_t)Ops::kSize * (kDlbTile + 2);
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaFuncSetAttribute(k_dlb<Ops>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr_set = true;
  }
  k_dlb<Ops><<<(unsigned)ntiles, kDlbTile, smem, L.stream>>>(
      ops, buf, n, rev, reinterpret_cast<char*>(state), ntiles);
  L.count("chunk_scan_dlb");
}

}  // namespace psk
