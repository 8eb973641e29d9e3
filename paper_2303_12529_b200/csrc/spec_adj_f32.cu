// Explicit instantiations of the adj spectral passes for float (parallel build units).
#include "spectral.cuh"

namespace lsb {
namespace spec {
template void a1_impl<float>(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
template void a2_impl<float>(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
template int finish_impl<float>(const Grid& g, const void* V0, const void* V1, double scale, double* out, const double* vp,
                double* dots, StopFlag stop, cudaStream_t s, int ix0, int ix1, const LoopTail* tail, int iy0,
                int iy1);
}  // namespace spec
}  // namespace lsb
