// Explicit instantiation of the FP64 DMMA GEMM for tile configuration CfgS.
#include "gemm_impl.cuh"
namespace ppc {
template void launch_cfg<CfgS>(const GemmParams&, dim3, bool, bool, bool, int, cudaStream_t);
}  // namespace ppc
