// Explicit instantiation of the FP64 DMMA GEMM for tile configuration CfgT16.
#include "gemm_impl.cuh"
namespace ppc {
template void launch_cfg<CfgT16>(const GemmParams&, dim3, bool, bool, bool, int, cudaStream_t);
}  // namespace ppc
