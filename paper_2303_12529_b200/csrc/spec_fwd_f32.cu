// Explicit instantiations of the fwd spectral passes for float (parallel build units).
#include "spectral.cuh"

namespace lsb {
namespace spec {
template void mask_fft_impl<float>(const Grid& g, const void* src, int kind, void* mhat, void* scratch, StopFlag stop,
                   cudaStream_t s);
template void f1_impl<float>(const Grid& g, const void* mhat, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
template void f2_impl<float>(const Grid& g, const SpecSet* sets, int nsets, double2* a0_out, StopFlag stop, cudaStream_t s);
}  // namespace spec
}  // namespace lsb
