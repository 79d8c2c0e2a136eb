// psk_tma.hpp -- host side of the TMA stage (psk_stage.cuh): one 3-D tensor
// map per model field, [row, L, nfull] = (one step's block padded to a 16-byte
// row) x (steps of a chunk) x (complete chunks), box {row, 1, kStageNT}.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "psk_common.cuh"
#include "psk_stage.cuh"

namespace psk {

inline PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// Fill `maps` for a staged walk over chunks of L steps, `nfull` of them
// complete.  A field is staged when its per-step blocks are whole 16-byte
// rows, or dense blocks of 4 / 8 bytes grouped 16 / bytes steps per row (L a
// multiple of that); any other non-broadcast field (a grouped field viewed
// at an odd step offset, as the PTFS backward pass's shifted model is) is
// read from global memory by the kernels.  Returns 0, or 9 when the TMA
// encoder is unavailable or rejects a map.
// L2 promotion of the staged boxes (experiment knobs for the ncu traffic
// check, 0..3 = none / 64 / 128 / 256 bytes): PSK_TMA_L2PROMO for rows of 64
// bytes and more (default 256), PSK_TMA_L2PROMO_SMALL for smaller rows
// (default none).  A promoted 256-byte line holds 8-16 steps of a 16/32-byte
// field of ONE chunk; the walk needs them over ~50 us, by which time ~300 MB
// have streamed through the 126 MB L2, so most of the promotion is evicted
// unused (profiles/r01_v4: finish reads 8.36 GB for 6.98 GB of inputs with
// 256 B everywhere; small rows unpromoted: 4.72 vs 4.89 ms per PRTS).
inline CUtensorMapL2promotion stage_l2_promotion(int row) {
  static const int big = [] {
    const char* v = std::getenv("PSK_TMA_L2PROMO");
    const int i = v ? std::atoi(v) : 3;
    return i < 0 || i > 3 ? 3 : i;
  }();
  static const int small = [] {
    const char* v = std::getenv("PSK_TMA_L2PROMO_SMALL");
    const int i = v ? std::atoi(v) : 0;
    return i < 0 || i > 3 ? 3 : i;
  }();
  return static_cast<CUtensorMapL2promotion>(row >= 64 ? big : small);
}

template <typename S, int NX, int NY>
int make_stage_maps(const ModelView<S>& m, long long L, long long nfull, StageMaps& maps) {
  using In = FilterTma<S, NX, NY>;
  const S* base[7] = {m.f, m.u, m.q, m.h, m.d, m.r, m.y};
  const long long stride[7] = {m.sf, m.su, m.sq, m.sh, m.sd, m.sr, m.sy};
  maps.tx = 0;
  for (int f = 0; f < 7; ++f) {
    maps.use[f] = 0;
    maps.grp[f] = 1;
    if (stride[f] == 0 || nfull <= 0) continue;  // broadcast: read from global
    auto enc = tma_encoder();
    if (!enc) return 9;
    const int row = In::row(f);
    const int bytes = (f == 0 || f == 2) ? NX * NX * (int)sizeof(S)
                      : f == 1           ? NX * (int)sizeof(S)
                      : f == 3           ? NY * NX * (int)sizeof(S)
                      : f == 5           ? NY * NY * (int)sizeof(S)
                                         : NY * (int)sizeof(S);
    const unsigned long long pitch = (unsigned long long)stride[f] * sizeof(S);
    const bool aligned = reinterpret_cast<uintptr_t>(base[f]) % 16 == 0;
    long long g = 1;  // steps per row
    if (aligned && pitch % 16 == 0 && pitch >= (unsigned long long)row) {
      g = 1;
    } else if (aligned && bytes < 16 && 16 % bytes == 0 && pitch == (unsigned long long)bytes &&
               L % (16 / bytes) == 0) {
      g = 16 / bytes;  // dense small blocks: rows of g consecutive steps
    } else {
      continue;  // not stageable (a grouped field at an odd step offset): global loads
    }
    const unsigned long long rpitch = g == 1 ? pitch : 16;  // bytes between rows
    cuuint64_t dims[3] = {(cuuint64_t)(row / sizeof(S)), (cuuint64_t)(L / g),
                          (cuuint64_t)nfull};
    cuuint64_t strides[2] = {(cuuint64_t)rpitch, (cuuint64_t)(pitch * (unsigned long long)L)};
    cuuint32_t box[3] = {(cuuint32_t)(row / sizeof(S)), 1, (cuuint32_t)kStageNT};
    cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapSwizzle sw = row == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : row == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : row == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                              : CU_TENSOR_MAP_SWIZZLE_NONE;
    const CUresult r =
        enc(&maps.m[f],
            sizeof(S) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
            3, const_cast<S*>(base[f]), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            stage_l2_promotion(row), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 9;
    maps.use[f] = 1;
    maps.grp[f] = (int)g;
    maps.tx += (unsigned)(row * kStageNT);
  }
  return 0;
}

// The filter finish's egl store map (EglStore): box {kStageNT chunks, ES
// components} of the [ecap, ES * L] egl tensor, staged in the first ES *
// kStageNT scalars of a consumed input stage (F, u, Q -- read at the start of
// a step) -- only where that region ends before H's box.  FP32 only: the
// extra block barrier per step (the element rows span every chunk's input
// rows) costs FP64 more than the saved stores (same box, 2^24: FP64 finish
// 1.983 -> 2.018 ms, FP32 1.016 -> 0.9996 ms; profiles/r02_v4/small_t.txt)
template <typename S, int NX, int NY>
int make_egl_store_map(S* egl, long long ecap, long long L, EglStore& em) {
  using In = FilterTma<S, NX, NY>;
  constexpr int ES = NX * NX + NX + NX * (NX + 1) / 2;
  em.use = 0;
  if (sizeof(S) != 4 || egl == nullptr || ES > 256 ||
      ES * kStageNT * (int)sizeof(S) > In::off(3) ||
      reinterpret_cast<uintptr_t>(egl) % 16 || (ecap * sizeof(S)) % 16)
    return 0;
  auto enc = tma_encoder();
  if (!enc) return 9;
  cuuint64_t dims[2] = {(cuuint64_t)ecap, (cuuint64_t)(ES * L)};
  cuuint64_t strides[1] = {(cuuint64_t)(ecap * sizeof(S))};
  cuuint32_t box[2] = {(cuuint32_t)kStageNT, (cuuint32_t)ES};
  cuuint32_t es[2] = {1, 1};
  if (enc(&em.map, sizeof(S) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
          2, egl, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 9;
  em.use = 1;
  return 0;
}

// Tensor maps of the smoother finish: the chunk-interleaved per-step
// elements egl[(j * ES + comp) * ecap + c] as a 2-D tensor [ecap, ES * L]
// (box {32, ES}) and the outputs mean[T][NX], cov[T][NX][NX] as 3-D tensors
// [row, L, nfull] (box {row, 1, 32}).  Rows that are not whole 16-byte units
// (odd NX in FP64, ...) are stored directly by the kernel (store = 0).
template <typename S, int NX>
int make_smooth_maps(const S* egl, long long ecap, long long L, long long nfull, S* mean,
                     S* cov, SmoothMaps& maps) {
  using Tm = SmoothTma<S, NX>;
  auto enc = tma_encoder();
  if (!enc) return 9;
  const CUtensorMapDataType dt =
      sizeof(S) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  {
    cuuint64_t dims[2] = {(cuuint64_t)ecap, (cuuint64_t)(Tm::ES * L)};
    cuuint64_t strides[1] = {(cuuint64_t)(ecap * sizeof(S))};
    cuuint32_t box[2] = {32, (cuuint32_t)Tm::ES};
    cuuint32_t es[2] = {1, 1};
    if (enc(&maps.egl, dt, 2, const_cast<S*>(egl), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 9;
  }
  maps.store = 0;
  const int mrow = NX * (int)sizeof(S), crow = NX * NX * (int)sizeof(S);
  if (nfull <= 0 || mrow % 16 || crow % 16 || crow > 256 * (int)sizeof(S) ||
      reinterpret_cast<uintptr_t>(mean) % 16 || reinterpret_cast<uintptr_t>(cov) % 16)
    return 0;
  auto out_map = [&](CUtensorMap* map, S* base, int row) {
    cuuint64_t dims[3] = {(cuuint64_t)(row / sizeof(S)), (cuuint64_t)L, (cuuint64_t)nfull};
    cuuint64_t strides[2] = {(cuuint64_t)row, (cuuint64_t)row * (cuuint64_t)L};
    cuuint32_t box[3] = {(cuuint32_t)(row / sizeof(S)), 1, 32};
    cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapSwizzle sw = row == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : row == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : row == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                              : CU_TENSOR_MAP_SWIZZLE_NONE;
    return enc(map, dt, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
  };
  if (!out_map(&maps.mean, mean, mrow) || !out_map(&maps.cov, cov, crow)) return 9;
  maps.store = 1;
  return 0;
}

}  // namespace psk
