// psk_fast_f32.cu -- float instantiations of the fast path (split per dtype
// so the two halves compile in parallel).
#include "psk_fast_impl.cuh"
#include "psk_wide_impl.cuh"

namespace psk {
template bool fast_supported<float>(int, int);
template int fast_run<float>(ExactLaunch&, const ModelView<float>&, const FastArgs&, float*, float*,
                          void* (*)(size_t, void*), void*);
template int fast_shard_phase<float>(ExactLaunch&, const ModelView<float>&, const FastArgs&, int,
                                  void**, float*, float*, const float*, float*,
                                  void* (*)(size_t, void*), void*, const float*, const float*);
template void fast_shard_release<float>(void*);
template int fast_ptfs2<float>(ExactLaunch&, const ModelView<float>&, int, ExactLaunch&,
                            const ModelView<float>&, int, const FastArgs&, float*, float*,
                            void* (*)(size_t, void*), void*, void* (*)(size_t, void*), void*);
template int fast_fold<float>(ExactLaunch&, int, int, const float*, int, float*);
template int wide::wide_run<float>(ExactLaunch&, const ModelView<float>&, const FastArgs&, float*,
                               float*, void* (*)(size_t, void*), void*);
template <>
int wide_run<float>(ExactLaunch& L, const ModelView<float>& m, const FastArgs& a, float* mean,
                   float* cov, void* (*alloc)(size_t, void*), void* actx) {
  if (a.tile) {
    const int st = tile_run<float>(L, m, a, mean, cov, alloc, actx);
    if (st != -1) return st;
  }
  return wide::wide_run<float>(L, m, a, mean, cov, alloc, actx);
}
}  // namespace psk
