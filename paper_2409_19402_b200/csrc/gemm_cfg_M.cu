// Explicit instantiation of the FP64 DMMA GEMM for tile configuration CfgM.
#include "gemm_impl.cuh"
namespace ppc {
template void launch_cfg<CfgM>(const GemmParams&, dim3, bool, bool, bool, int, cudaStream_t);
}  // namespace ppc
