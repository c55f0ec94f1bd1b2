#pragma once
// Projection transforms (proj/include/projprod/transforms.hpp).
#include <cstdint>
#include <optional>

#include "projprod/tensor.hpp"

namespace projprod {

enum class TransformKind { Identity, RandomOrthogonal, Dct, DataDependent, Haar, Custom };

struct Transform {
    Matrix Q;  // n3 x p, orthonormal columns
    TransformKind kind = TransformKind::Custom;
    std::optional<std::uint64_t> seed;
    double scale = 1.0;  // weight c of a scaled basis W = cQ (applied by the star product)
    bool completed_basis = false;
    Index n3() const { return Q.rows(); }
    Index p() const { return Q.cols(); }
};

Transform identity_transform(Index n3, Index p);
Transform random_orthogonal_transform(Index n3, Index p, std::uint64_t seed);
Transform dct_transform(Index n3, Index p);
// Q = U3(:,1:p) of the mode-3 unfolding; on the device via a deterministic
// Gram SYRK + top-p symmetric eigensolve (bitwise repeatable).
Transform data_dependent_transform(const Tensor3& A, Index p);
Transform haar_transform(Index n3, Index p);
Transform custom_transform(Matrix Q, double scale = 1.0);
Matrix complement_basis(const Transform& T);
// ||A x_3 (I - QQ^T)||_F, fused on the device (no N x n3 temporary).
double projection_error(const Tensor3& A, const Transform& T);

}  // namespace projprod
