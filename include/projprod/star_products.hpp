#pragma once
// Projected tensor-tensor product (proj/include/projprod/star_products.hpp).
#include <optional>

#include "projprod/transforms.hpp"

namespace projprod {

struct StarContext {
    Transform transform;
    std::optional<Matrix> complement;  // n3 x (n3 - p)
    explicit StarContext(Transform T) : transform(std::move(T)) {}
    static StarContext with_complement(Transform T);
};

// [(A x3 M) facewise (B x3 M)] x3 M^{-1} for an invertible n3 x n3 M
// (degenerate_input_error when M is numerically singular).
Tensor3 star_m_product(const Tensor3& A, const Tensor3& B, const Matrix& M);
// ((A x3 Q^T) facewise (B x3 Q^T)) x3 Q, times the context's scale.
Tensor3 star_q_product(const Tensor3& A, const Tensor3& B, const StarContext& ctx);
// The m x m x n3 identity of the projected algebra (divided by the scale).
Tensor3 star_q_identity(Index m, const StarContext& ctx);
// Slice-wise transpose in the transform domain.
Tensor3 star_q_transpose(const Tensor3& A, const StarContext& ctx);

}  // namespace projprod
