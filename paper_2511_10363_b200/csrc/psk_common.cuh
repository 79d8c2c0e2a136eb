// psk_common.cuh -- device-side views shared by the fast and exact paths.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace psk {

// device error bits (mapped to psk status codes by the host)
enum : unsigned { kErrNotPD = 1u, kErrSingular = 2u };

// Device view of psk_model (include/psk.h): per-field base + step stride in
// scalars (0 = broadcast).  Index convention of lgssm.hpp:5-8.
template <typename S>
struct ModelView {
  const S *f, *u, *q, *h, *d, *r, *y;
  long long sf, su, sq, sh, sd, sr, sy;
  const S *m0, *p0;
  long long t;
  int nx, ny;
  // time sharding (paper_2511_10363_b200/distributed.py): local step 0
  // absorbs the prior only in the first shard; `last_step` is the local index
  // of the series' last step T-1 (-1 when this shard does not contain it, in
  // which case f/u/q carry one extra transition at local index t)
  int prior_first;
  long long last_step;
  __device__ __forceinline__ const S* F(long long k) const { return f + k * sf; }
  __device__ __forceinline__ const S* U(long long k) const { return u + k * su; }
  __device__ __forceinline__ const S* Q(long long k) const { return q + k * sq; }
  __device__ __forceinline__ const S* H(long long k) const { return h + k * sh; }
  __device__ __forceinline__ const S* D(long long k) const { return d + k * sd; }
  __device__ __forceinline__ const S* R(long long k) const { return r + k * sr; }
  __device__ __forceinline__ const S* Y(long long k) const { return y + k * sy; }
};

// Structure-of-arrays element buffer: component c of slot i at
// p[c * cap + i] (coalesced across consecutive slots).  `rev` implements the
// reference's Reversed<E> adapter (scan.hpp:149-177): logical slot i lives at
// physical cap-1-i ... of the logical size `n`.
// Storage slot of chunk c in a chunk-element buffer (SoA, one slot per
// chunk).  per = 0: chunk order.  per >= 1 (buffers scanned by the decoupled
// look-back, psk_dlb.cuh): slots follow the SCAN order (reversed for reverse
// scans) and, inside each tile of kOrderNT * per elements, element
// r = t per + j of the tile sits at j kOrderNT + t -- the per consecutive
// elements of look-back thread t are then coalesced across the threads.
constexpr int kOrderNT = 128;  // == kDlbThreads
struct ChunkOrder {
  long long n;  // chunks
  int per;
  int rev;
  __host__ __device__ __forceinline__ long long at(long long c) const {
    if (per == 0) return c;
    const long long g = rev ? n - 1 - c : c;
    const long long tile = (long long)kOrderNT * per;
    const long long b = g / tile * tile, r = g - b;
    return b + (r % per) * kOrderNT + r / per;
  }
  // slots a buffer in this order needs
  __host__ __device__ long long cap() const {
    if (per == 0) return n;
    const long long tile = (long long)kOrderNT * per;
    return (n + tile - 1) / tile * tile;
  }
};

template <typename S>
struct ElemBuf {
  S* p;
  long long cap;  // physical slots (component stride)
  long long n;    // logical size
  int rev;
  __device__ __forceinline__ long long phys(long long i) const {
    return rev ? n - 1 - i : i;
  }
};

// One level of a level-by-level scan (the reference's Launch per level,
// scan.hpp:198-444).  Buffers: 0 = a (main), 1 = aux/orig/arena, 2 = tmp.
enum LevelKind : int {
  kLvSeqChain = 0,   // a[i+1] = a[i] (x) a[i+1], i = 0..n-2, one thread
  kLvHS = 1,         // nxt[nb+i] = i>=delta ? cur[cb+i-delta] (x) cur[cb+i] : cur[cb+i]
  kLvCopy = 2,       // dst[db+i] = src[sb+i], i < count
  kLvUp = 3,         // a[m d2 + d2-1] = a[m d2 + d1-1] (x) a[m d2 + d2-1]
  kLvIdentity = 4,   // a[idx] = e
  kLvBlDown = 5,     // t=a_j; a_j=a_k; a_k=a_k (x) t   (tmp[m])
  kLvBlFinal = 6,    // a[i] = a[i] (x) orig[i]
  kLvLafiDown = 7,   // a[j] = a[i] (x) a[j], i=(m+1)d2-1, j=i+d1
  kLvSgReduce = 8,   // arena[do+m] = src[so+2m] (x) src[so+2m+1]
  kLvSgDist = 9,     // distribute (scan.hpp:419-444)
};

struct LevelDesc {
  int kind;
  int bufA, bufB, bufC;  // buffer ids used by the level (meaning per kind)
  long long count;       // number of iterations
  long long p0, p1, p2;  // kind-specific parameters (offsets / deltas)
};

}  // namespace psk
