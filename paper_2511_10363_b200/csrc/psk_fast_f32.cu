// psk_fast_f32.cu -- float instantiations of the fast path (split per
// dtype so the two halves compile in parallel).
#include "psk_fast_impl.cuh"

namespace psk {
template bool fast_supported<float>(int, int);
template int fast_run<float>(ExactLaunch&, const ModelView<float>&, const FastArgs&,
                          float*, float*, void* (*)(size_t, void*), void*);
}  // namespace psk
