// psk_tile_f32.cu -- float instantiations of the register-tiled warp kernels
// (psk_tile_impl.cuh), a translation unit of their own so they compile in
// parallel with the rest of the fast path.
#include "psk_tile_impl.cuh"

namespace psk {
template <>
int tile_run<float>(ExactLaunch& L, const ModelView<float>& m, const FastArgs& a, float* mean,
                 float* cov, void* (*alloc)(size_t, void*), void* actx) {
  return tile::tile_run<float>(L, m, a, mean, cov, alloc, actx);
}
}  // namespace psk
