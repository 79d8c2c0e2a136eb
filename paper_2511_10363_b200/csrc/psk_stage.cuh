// psk_stage.cuh -- TMA staging of the per-step model blocks into shared
// memory (cp.async.bulk.tensor + mbarrier), double-buffered.
//
// Every fast-path thread walks its own chunk of L consecutive steps; a CTA of
// kStageNT threads owns kStageNT consecutive chunks, so at walk position j it
// needs step j of each of them: kStageNT blocks spaced L steps apart in every
// field array.  Viewed as a 3-D tensor [row, L, chunks] (row = one step's
// block, padded to 16 bytes), that set is ONE tensor-map box {row, 1,
// kStageNT} per field -- seven TMA instructions fetch a whole step of the
// CTA.  Measured on the pure chunk walk (psk_membench.cu, profiles/r01_v2):
// TMA boxes 6.4-7.1 TB/s against 3.5-4.0 TB/s for warp-cooperative LDGSTS,
// 1.5-1.9 TB/s for per-thread loads and 2.2 TB/s for per-thread bulk copies.
//
// Box rows are swizzled by the TMA unit (128/64/32-byte modes for 128/64/
// 32-byte rows) so that each thread's 16-byte reads of its own row are
// bank-conflict-free; rows of other widths are unswizzled (odd multiples of
// 16 bytes are conflict-free as they are).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "psk_mat.cuh"

namespace psk {

constexpr int kStageNT = 128;  // threads (= chunks) per CTA of a staged walk

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "PSK_WAIT: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra PSK_WAIT;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(b))
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2,
                                             const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          map),
      "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1,
                                             const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          map),
      "r"(c0), "r"(c1), "r"(smem_u32(src))
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// wait until at most N committed bulk groups still READ shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// One staged field: BYTES per step, row = BYTES rounded up to 16, box of
// kStageNT rows at byte OFF (1024-aligned) of a stage.
template <int OFF, int BYTES>
struct TField {
  static constexpr int bytes = BYTES;
  static constexpr int row = (BYTES + 15) / 16 * 16;
  static constexpr int swz = row == 128 ? 3 : (row == 64 ? 2 : (row == 32 ? 1 : 0));
  static constexpr int off = OFF;
  static constexpr int end = OFF + (row * kStageNT + 1023) / 1024 * 1024;
};
// byte offset of 16-byte chunk c of row r inside the field's box (the TMA
// swizzle: address bits [4, 4+swz) ^= bits [7, 7+swz))
template <class F>
__device__ __forceinline__ int tma_off(int r, int c) {
  const int a = r * F::row + c * 16;
  return a ^ (((a >> 7) & ((1 << F::swz) - 1)) << 4);
}
// this thread's block of a staged field as a row-major R x C matrix
// `sub`: byte offset of this step's block inside a row that packs several
// steps of a small field (grouped rows, see StageMaps::grp); 0 otherwise.
template <class F, typename S, int R, int C>
__device__ __forceinline__ Mat<S, R, C> tma_get(const unsigned char* stage, int t, int sub = 0) {
  static_assert(R * C * (int)sizeof(S) == F::bytes, "field size");
  Mat<S, R, C> m;
  S* o = &m.a[0][0];
  constexpr int per = 16 / sizeof(S);
  constexpr int n = R * C;
#pragma unroll
  for (int c = 0; c < (n + per - 1) / per; ++c) {
    const unsigned char* p = stage + F::off + tma_off<F>(t, c) + sub;
    if ((c + 1) * per <= n) {
      const float4 v = *reinterpret_cast<const float4*>(p);
      const S* vs = reinterpret_cast<const S*>(&v);
#pragma unroll
      for (int j = 0; j < per; ++j) o[c * per + j] = vs[j];
    } else {
#pragma unroll
      for (int j = 0; j < per; ++j)
        if (c * per + j < n) o[c * per + j] = reinterpret_cast<const S*>(p)[j];
    }
  }
  return m;
}

// The staged filter inputs (F, u, Q, H, d, R, y) of one step of a CTA
template <typename S, int NX, int NY>
struct FilterTma {
  static constexpr int s = sizeof(S);
  using F = TField<0, NX * NX * s>;
  using u = TField<F::end, NX * s>;
  using Q = TField<u::end, NX * NX * s>;
  using H = TField<Q::end, NY * NX * s>;
  using d = TField<H::end, NY * s>;
  using R = TField<d::end, NY * NY * s>;
  using y = TField<R::end, NY * s>;
  static constexpr int stage = y::end;  // bytes of one stage (1024-aligned)
  __host__ __device__ static constexpr int off(int f) {
    return f == 0 ? F::off : f == 1 ? u::off : f == 2 ? Q::off : f == 3 ? H::off
         : f == 4 ? d::off : f == 5 ? R::off : y::off;
  }
  __host__ __device__ static constexpr int row(int f) {
    return f == 0 ? F::row : f == 1 ? u::row : f == 2 ? Q::row : f == 3 ? H::row
         : f == 4 ? d::row : f == 5 ? R::row : y::row;
  }
  // dynamic shared memory of a walk with `ns` stages (steps in flight + 1),
  // + alignment slack and the mbarriers
  __host__ __device__ static constexpr int smem_n(int ns) { return ns * stage + 1024 + 64; }
  static constexpr int smem = smem_n(2);
  // stages of the filter finish: an FP32 step is cheaper and its stage half
  // as large, so two stages leave the finish waiting on TMA latency; three
  // (28 KB each at nx = 4) still fit its 2 CTAs per SM (register-bound).
  // The reduce keeps two (3 CTAs/SM in FP32: measured faster than 2 x 3
  // stages; 4 stages fit only 1 CTA/SM, 2x slower).  FP64: two 53 KB stages.
  // FP32 takes a fourth stage where two CTAs still fit (nx = 4, ny <= 2)
  // (2 stages at 3 CTAs/SM -- 168 registers, no spills -- measured 1.18 vs
  // 1.115 ms, same box)
  static constexpr int finish_stages =
      sizeof(S) == 8 ? 2 : (2 * smem_n(4) <= 220 * 1024 ? 4 : 3);
  static constexpr int finish_ctas = 2;
};

// this thread's row of a staged field <- a row-major R x C matrix (the
// inverse of tma_get, for TMA stores)
template <class F, typename S, int R, int C>
__device__ __forceinline__ void tma_put(unsigned char* stage, int t, const Mat<S, R, C>& m) {
  static_assert(R * C * (int)sizeof(S) == F::bytes && F::bytes % 16 == 0, "field size");
  const S* o = &m.a[0][0];
  constexpr int per = 16 / sizeof(S);
#pragma unroll
  for (int c = 0; c < R * C / per; ++c) {
    float4 v;
    S* vs = reinterpret_cast<S*>(&v);
#pragma unroll
    for (int j = 0; j < per; ++j) vs[j] = o[c * per + j];
    *reinterpret_cast<float4*>(stage + F::off + tma_off<F>(t, c)) = v;
  }
}

// TMA store of the PRTS filter finish's per-step smoothing elements: the
// chunk-interleaved egl buffer as a 2-D tensor [ecap, ES * L] written one
// walk position of the CTA's 128 chunks at a time (box {kStageNT, ES}) from
// the consumed input stage (kernel parameter; use = 0: plain stores).
struct EglStore {
  CUtensorMap map;
  int use;
};

// Tensor maps of the seven model fields for one staged launch (kernel
// parameter; `use[f]` = 0 for a broadcast field, read straight from global).
struct StageMaps {
  CUtensorMap m[7];
  int use[7];
  // steps per 16-byte row: a field whose per-step block is 4 or 8 bytes and
  // dense (e.g. d, y at ny = 2 in FP32) is viewed as rows of 16 / bytes
  // consecutive steps, so it is staged in place instead of re-pitched; the
  // box of walk position j is row j / grp, the step's block at (j % grp)
  int grp[7];
  unsigned tx;  // bytes one stage receives (sum of the used boxes)
};

// Smoother finish of a warp (32 chunks): TMA loads of the per-step smoothing
// elements (2-D box {32 chunks, ES components} of the chunk-interleaved
// buffer) and TMA stores of the smoothed (mean, cov) rows (3-D boxes {row,
// 1, 32} of the output arrays), both double-buffered.
struct SmoothMaps {
  CUtensorMap egl;
  CUtensorMap mean;
  CUtensorMap cov;
  int store;  // 0: rows are not whole 16-byte units -> plain stores
};
template <typename S, int NX>
struct SmoothTma {
  static constexpr int ES = NX * NX + NX + NX * (NX + 1) / 2;  // EglLayout<NX>::size
  static constexpr int egl_box = 32 * ES * (int)sizeof(S);
  static constexpr int egl_stage = (egl_box + 1023) / 1024 * 1024;
  using Mean = TField<0, NX * (int)sizeof(S)>;  // rows of a 32-row box
  static constexpr int mean_stage = (Mean::row * 32 + 1023) / 1024 * 1024;
  using Cov = TField<0, NX * NX * (int)sizeof(S)>;
  static constexpr int cov_stage = (Cov::row * 32 + 1023) / 1024 * 1024;
  // element stages of the per-warp pipeline: four (3 boxes in flight per
  // warp; FP64 2 CTAs/SM, FP32 4) -- measured against 2 and 3 stages:
  // FP64 1.165 / 1.133 / 1.116 ms, FP32 0.671 (2) / 0.629 ms (4) at 2^24
  // FP32 boxes are half as large: seven stages (3 CTAs/SM at nx = 4) keep
  // about as many bytes in flight per SM as FP64's four
  static constexpr int egl_nstage = sizeof(S) == 4 ? 7 : 4;
  // one warp: egl_nstage egl stages, 2 mean stages, 2 cov stages, mbarriers
  static constexpr int warp =
      egl_nstage * egl_stage + 2 * (mean_stage + cov_stage) + 1024;
};

}  // namespace psk
