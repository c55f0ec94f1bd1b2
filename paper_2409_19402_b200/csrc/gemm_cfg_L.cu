// Explicit instantiation of the FP64 DMMA GEMM for tile configuration CfgL.
#include "gemm_impl.cuh"
namespace ppc {
template void launch_cfg<CfgL>(const GemmParams&, dim3, bool, bool, bool, int, cudaStream_t);
}  // namespace ppc
