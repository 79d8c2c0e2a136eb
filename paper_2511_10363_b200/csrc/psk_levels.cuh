// psk_levels.cuh -- one generic kernel that executes a level of a
// level-by-level scan (the reference's one-Launch-per-level kernels,
// scan.hpp:198-444), parameterised by an element-operator policy `Ops`:
//   Ops::S                               scalar
//   ops.combine(dst, di, l, li, r, ri)   dst[di] = l[li] (x) r[ri] (physical)
//   ops.assign(dst, di, src, si)
//   ops.identity(dst, di)
// Operand order is flipped for reversed buffers (Reversed<E>::combine,
// scan.hpp:164-167).  Iterations of one level write disjoint slots, as the
// reference's WriteSetRecorderBackend checks (backend.hpp:134-151).
#pragma once
#include "psk_common.cuh"

namespace psk {

template <class Ops>
struct Bufs3 {
  ElemBuf<typename Ops::S> b[3];
};

template <class Ops>
__device__ __forceinline__ void h_combine(const Ops& ops,
                                          const ElemBuf<typename Ops::S>& dst,
                                          long long di,
                                          const ElemBuf<typename Ops::S>& l,
                                          long long li,
                                          const ElemBuf<typename Ops::S>& r,
                                          long long ri) {
  if (!dst.rev)
    ops.combine(dst, dst.phys(di), l, l.phys(li), r, r.phys(ri));
  else
    ops.combine(dst, dst.phys(di), r, r.phys(ri), l, l.phys(li));
}
template <class Ops>
__device__ __forceinline__ void h_assign(const Ops& ops,
                                         const ElemBuf<typename Ops::S>& dst,
                                         long long di,
                                         const ElemBuf<typename Ops::S>& src,
                                         long long si) {
  ops.assign(dst, dst.phys(di), src, src.phys(si));
}

// UNIT = threads per iteration: 1 (one thread per combine, register-resident
// operators) or 32 (one warp per combine: the warp-cooperative operators of
// psk_wide.cuh; every lane of the warp runs the same iteration).
template <class Ops, int UNIT = 1>
__global__ void __launch_bounds__(128) k_level(Ops ops, Bufs3<Ops> bufs,
                                               LevelDesc d) {
  const long long stride = (long long)gridDim.x * blockDim.x / UNIT;
  for (long long m = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / UNIT;
       m < d.count; m += stride) {
    switch (d.kind) {
      case kLvSeqChain: {
        if (m != 0) return;
        const auto& a = bufs.b[0];
        for (long long i = 0; i < d.count; ++i) h_combine(ops, a, i + 1, a, i, a, i + 1);
        return;
      }
      case kLvHS: {
        const auto& cur = bufs.b[d.bufA];
        const auto& nxt = bufs.b[d.bufB];
        const long long cb = d.p0, nb = d.p1, delta = d.p2;
        if (m >= delta)
          h_combine(ops, nxt, nb + m, cur, cb + m - delta, cur, cb + m);
        else
          h_assign(ops, nxt, nb + m, cur, cb + m);
        break;
      }
      case kLvCopy:
        h_assign(ops, bufs.b[d.bufA], d.p0 + m, bufs.b[d.bufB], d.p1 + m);
        break;
      case kLvUp: {
        const auto& a = bufs.b[0];
        const long long j = m * d.p1 + d.p0 - 1, kk = m * d.p1 + d.p1 - 1;
        h_combine(ops, a, kk, a, j, a, kk);
        break;
      }
      case kLvIdentity:
        if (m == 0) ops.identity(bufs.b[d.bufA], bufs.b[d.bufA].phys(d.p0));
        break;
      case kLvBlDown: {
        const auto& a = bufs.b[0];
        const auto& t = bufs.b[d.bufB];
        const long long j = m * d.p1 + d.p0 - 1, kk = m * d.p1 + d.p1 - 1;
        h_assign(ops, t, m, a, j);
        h_assign(ops, a, j, a, kk);
        h_combine(ops, a, kk, a, kk, t, m);
        break;
      }
      case kLvBlFinal:
        h_combine(ops, bufs.b[0], m, bufs.b[0], m, bufs.b[d.bufB], m);
        break;
      case kLvLafiDown: {
        const auto& a = bufs.b[0];
        const long long i = (m + 1) * d.p1 - 1, j = i + d.p0;
        h_combine(ops, a, j, a, i, a, j);
        break;
      }
      case kLvSgReduce: {
        const auto& dst = bufs.b[d.bufA];
        const auto& src = bufs.b[d.bufB];
        h_combine(ops, dst, d.p0 + m, src, d.p1 + 2 * m, src, d.p1 + 2 * m + 1);
        break;
      }
      case kLvSgDist: {
        if (m == 0) break;
        const auto& dst = bufs.b[d.bufA];
        const auto& par = bufs.b[d.bufB];
        if ((m & 1) == 0)
          h_combine(ops, dst, d.p0 + m, par, d.p1 + m / 2 - 1, dst, d.p0 + m);
        else
          h_assign(ops, dst, d.p0 + m, par, d.p1 + (m - 1) / 2);
        break;
      }
      default:
        break;
    }
  }
}

}  // namespace psk
