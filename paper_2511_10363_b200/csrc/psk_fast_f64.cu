// psk_fast_f64.cu -- double instantiations of the fast path (split per dtype
// so the two halves compile in parallel).
#include "psk_fast_impl.cuh"
#include "psk_wide_impl.cuh"

namespace psk {
template bool fast_supported<double>(int, int);
template int fast_run<double>(ExactLaunch&, const ModelView<double>&, const FastArgs&, double*, double*,
                          void* (*)(size_t, void*), void*);
template int fast_shard_phase<double>(ExactLaunch&, const ModelView<double>&, const FastArgs&, int,
                                  void**, double*, double*, const double*, double*,
                                  void* (*)(size_t, void*), void*, const double*, const double*);
template void fast_shard_release<double>(void*);
template int fast_ptfs2<double>(ExactLaunch&, const ModelView<double>&, int, ExactLaunch&,
                            const ModelView<double>&, int, const FastArgs&, double*, double*,
                            void* (*)(size_t, void*), void*, void* (*)(size_t, void*), void*);
template int fast_fold<double>(ExactLaunch&, int, int, const double*, int, double*);
template int wide::wide_run<double>(ExactLaunch&, const ModelView<double>&, const FastArgs&, double*,
                               double*, void* (*)(size_t, void*), void*);
template <>
int wide_run<double>(ExactLaunch& L, const ModelView<double>& m, const FastArgs& a, double* mean,
                   double* cov, void* (*alloc)(size_t, void*), void* actx) {
  if (a.tile) {
    const int st = tile_run<double>(L, m, a, mean, cov, alloc, actx);
    if (st != -1) return st;
  }
  return wide::wide_run<double>(L, m, a, mean, cov, alloc, actx);
}
}  // namespace psk
