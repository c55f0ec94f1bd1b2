// Large-problem eigensolver / slice SVD (Gram + Chebyshev-filtered subspace
// iteration + Rayleigh-Ritz polish). Placeholder until the path lands.
#include "internal.h"
#include "slice_svd.cuh"

namespace ppc {
void subspace_eig_top(const double*, int64_t, int64_t, int64_t, double*, double*, cudaStream_t) {
    fail(PPC_ARGUMENT, "subspace_eig_top: not available yet");
}
void subspace_svd(const double*, int64_t, int64_t, int64_t, int64_t, int64_t, double*, double*,
                  double*, double*, cudaStream_t) {
    fail(PPC_ARGUMENT, "subspace_svd: not available yet");
}
}  // namespace ppc
