// psk_fast_f64.cu -- double instantiations of the fast path (split per
// dtype so the two halves compile in parallel).
#include "psk_fast_impl.cuh"

namespace psk {
template bool fast_supported<double>(int, int);
template int fast_run<double>(ExactLaunch&, const ModelView<double>&, const FastArgs&,
                          double*, double*, void* (*)(size_t, void*), void*);
}  // namespace psk
