// psk_tile_f64.cu -- double instantiations of the register-tiled warp kernels
// (psk_tile_impl.cuh), a translation unit of their own so they compile in
// parallel with the rest of the fast path.
#include "psk_tile_impl.cuh"

namespace psk {
template <>
int tile_run<double>(ExactLaunch& L, const ModelView<double>& m, const FastArgs& a, double* mean,
                 double* cov, void* (*alloc)(size_t, void*), void* actx) {
  return tile::tile_run<double>(L, m, a, mean, cov, alloc, actx);
}
}  // namespace psk
