#pragma once
// Metrics on the hot path (proj/include/projprod/metrics.hpp:21).
#include "projprod/decompositions.hpp"
#include "projprod/tensor.hpp"

namespace projprod {

// ||A - Ahat||_F / ||A||_F; the reference tensor must be nonzero.
double relative_error(const Tensor3& A, const Tensor3& Ahat);
// relative_error(A, tsvdq_reconstruct(F)) without materializing the
// reconstruction (fused on the device).
double tsvdq_relative_error(const Tensor3& A, const TsvdqFactors& F);

}  // namespace projprod
