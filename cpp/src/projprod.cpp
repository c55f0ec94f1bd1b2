// The projprod C++ API (proj/include/projprod/*.hpp signatures) on top of the
// B200 engine's C-ABI (include/ppc.h). Host buffers are passed with
// loc = PPC_HOST; the engine stages them through HBM. Argument checks and
// messages follow the reference; ppc status codes become the reference's
// exception types.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ppc.h"
#include "projprod/decompositions.hpp"
#include "projprod/engine.hpp"
#include "projprod/io.hpp"
#include "projprod/errors.hpp"
#include "projprod/matrix_kernels.hpp"
#include "projprod/metrics.hpp"
#include "projprod/star_products.hpp"
#include "projprod/parallel.hpp"
#include "projprod/tensor.hpp"
#include "projprod/transforms.hpp"

namespace projprod {

void throw_status(int code, const char* message) {
    const std::string m = message ? message : "";
    switch (code) {
        case PPC_OK: return;
        case PPC_SHAPE: throw shape_error(m);
        case PPC_BOUNDS: throw bounds_error(m);
        case PPC_ARGUMENT: throw argument_error(m);
        case PPC_DEGENERATE: throw degenerate_input_error(m);
        case PPC_NUMERIC: throw numeric_error(m);
        case PPC_FORMAT: throw format_error(m);
        default: throw device_error(m);
    }
}

namespace {
inline void check(int rc) {
    if (rc) throw_status(rc, ppc_last_error());
}
std::string shape_str(const Tensor3& A) {
    return std::to_string(A.n1()) + "x" + std::to_string(A.n2()) + "x" + std::to_string(A.n3());
}
}  // namespace

// ------------------------------------------------------------------ Tensor3
Tensor3::Tensor3(Index n1, Index n2, Index n3) : n1_(n1), n2_(n2), n3_(n3) {  // tensor.cpp:20-28
    if (n1 < 1 || n2 < 1 || n3 < 1)
        throw shape_error("tensor extents must be positive, got " + std::to_string(n1) + "x" +
                          std::to_string(n2) + "x" + std::to_string(n3));
    buf_.assign(static_cast<std::size_t>(n1 * n2 * n3), 0.0);
}

Tensor3 Tensor3::from_slices(const std::vector<Matrix>& slices) {  // tensor.cpp:30-43
    if (slices.empty()) throw shape_error("from_slices: empty slice list");
    Tensor3 out(slices[0].rows(), slices[0].cols(), static_cast<Index>(slices.size()));
    for (Index k = 0; k < out.n3(); ++k) {
        const Matrix& S = slices[static_cast<std::size_t>(k)];
        if (S.rows() != out.n1() || S.cols() != out.n2())
            throw shape_error("from_slices: slice " + std::to_string(k) + " has mismatched shape");
        out.set_slice(k, S);
    }
    return out;
}

Matrix Tensor3::slice(Index k) const {
    Matrix m(n1_, n2_);
    std::copy(slice_data(k), slice_data(k) + n1_ * n2_, m.data());
    return m;
}

void Tensor3::set_slice(Index k, const Matrix& m) {
    if (m.rows() != n1_ || m.cols() != n2_) throw shape_error("set_slice: shape mismatch");
    std::copy(m.data(), m.data() + n1_ * n2_, slice_data(k));
}

Matrix Tensor3::tubes_view() const {
    Matrix m(n1_ * n2_, n3_);
    std::copy(buf_.begin(), buf_.end(), m.data());
    return m;
}

Matrix frontal_slice(const Tensor3& A, Index k) {
    if (k < 0 || k >= A.n3())
        throw bounds_error("frontal_slice: k=" + std::to_string(k) + " outside [0," +
                           std::to_string(A.n3()) + ")");
    return A.slice(k);
}

Vector tube(const Tensor3& A, Index i, Index j) {
    if (i < 0 || i >= A.n1() || j < 0 || j >= A.n2())
        throw bounds_error("tube: (" + std::to_string(i) + "," + std::to_string(j) + ") outside " +
                           shape_str(A));
    Vector v(A.n3());
    for (Index k = 0; k < A.n3(); ++k) v(k) = A(i, j, k);
    return v;
}

Matrix mode3_unfold(const Tensor3& A) { return A.tubes_view().transpose(); }

Tensor3 mode3_fold(const Matrix& U, Index n1, Index n2, Index n3) {
    if (U.rows() != n3 || U.cols() != n1 * n2)
        throw shape_error("mode3_fold: unfolding is " + std::to_string(U.rows()) + "x" +
                          std::to_string(U.cols()) + ", expected " + std::to_string(n3) + "x" +
                          std::to_string(n1 * n2));
    Tensor3 out(n1, n2, n3);
    const Matrix t = U.transpose();
    std::copy(t.data(), t.data() + t.size(), out.data());
    return out;
}

Tensor3 mode3_product(const Tensor3& A, const Matrix& M) {  // tensor.cpp:139-147
    if (M.cols() != A.n3())
        throw shape_error("mode3_product: M has " + std::to_string(M.cols()) + " cols, tensor n3=" +
                          std::to_string(A.n3()));
    Tensor3 out(A.n1(), A.n2(), M.rows());
    check(ppc_mode3_product(A.data(), A.n1(), A.n2(), A.n3(), M.data(), M.rows(), 0, out.data(),
                            PPC_HOST));
    return out;
}

Matrix mode_unfold(const Tensor3& A, int mode) {  // tensor.cpp:87-107 (host-side layout)
    const Index n1 = A.n1(), n2 = A.n2(), n3 = A.n3();
    if (mode == 3) return mode3_unfold(A);
    if (mode == 1) {  // n1 x (n2 n3), column j + k n2: the buffer itself
        Matrix out(n1, n2 * n3);
        std::copy(A.data(), A.data() + A.size(), out.data());
        return out;
    }
    if (mode == 2) {  // n2 x (n1 n3), column i + k n1: slice-wise transposes
        Matrix out(n2, n1 * n3);
        for (Index k = 0; k < n3; ++k)
            for (Index i = 0; i < n1; ++i)
                for (Index j = 0; j < n2; ++j) out(j, i + k * n1) = A(i, j, k);
        return out;
    }
    throw argument_error("mode_unfold: mode must be 1, 2 or 3, got " + std::to_string(mode));
}

Tensor3 mode_product(const Tensor3& A, const Matrix& M, int mode) {  // tensor.cpp:109-137
    if (mode == 3) return mode3_product(A, M);
    if (mode != 1 && mode != 2)
        throw argument_error("mode_product: mode must be 1, 2 or 3, got " + std::to_string(mode));
    const Index ext = mode == 1 ? A.n1() : A.n2();
    if (M.cols() != ext)
        throw shape_error("mode_product(" + std::to_string(mode) + "): M has " + std::to_string(M.cols()) +
                          " cols, tensor n" + std::to_string(mode) + "=" + std::to_string(ext));
    Tensor3 out(mode == 1 ? M.rows() : A.n1(), mode == 2 ? M.rows() : A.n2(), A.n3());
    check(ppc_mode_product(A.data(), A.n1(), A.n2(), A.n3(), M.data(), M.rows(), mode, out.data(), PPC_HOST));
    return out;
}

Tensor3 facewise_product(const Tensor3& A, const Tensor3& B) {  // tensor.cpp:149-156
    if (A.n2() != B.n1() || A.n3() != B.n3())
        throw shape_error("facewise_product: " + shape_str(A) + " vs " + shape_str(B));
    Tensor3 out(A.n1(), B.n2(), A.n3());
    check(ppc_facewise_product(A.data(), A.n1(), A.n2(), A.n3(), B.data(), B.n2(), out.data(),
                               PPC_HOST));
    return out;
}

double frobenius_norm(const Tensor3& A) {
    double out = 0.0;
    check(ppc_frobenius_norm(A.data(), A.size(), &out, PPC_HOST));
    return out;
}

Tensor3 operator+(const Tensor3& A, const Tensor3& B) {
    if (!A.same_shape(B)) throw shape_error("tensor sum: " + shape_str(A) + " vs " + shape_str(B));
    Tensor3 out = A;
    for (Index i = 0; i < out.size(); ++i) out.data()[i] += B.data()[i];
    return out;
}

Tensor3 operator-(const Tensor3& A, const Tensor3& B) {
    if (!A.same_shape(B))
        throw shape_error("tensor difference: " + shape_str(A) + " vs " + shape_str(B));
    Tensor3 out = A;
    for (Index i = 0; i < out.size(); ++i) out.data()[i] -= B.data()[i];
    return out;
}

Tensor3 operator*(double c, const Tensor3& A) {
    Tensor3 out = A;
    for (Index i = 0; i < out.size(); ++i) out.data()[i] *= c;
    return out;
}

// ------------------------------------------------------------ matrix kernels
SvdResult truncated_svd(const Matrix& A, Index k) {  // matrix_kernels.cpp:39-46
    if (A.rows() < 1 || A.cols() < 1) throw shape_error("svd: empty matrix");
    const Index r = std::min(A.rows(), A.cols());
    if (k < 1 || k > r)
        throw argument_error("truncated_svd: k=" + std::to_string(k) + " outside [1," +
                             std::to_string(r) + "]");
    SvdResult out{Matrix(A.rows(), k), Vector(k), Matrix(A.cols(), k)};
    check(ppc_svd_batched(A.data(), A.rows(), A.cols(), 1, k, out.U.data(), out.s.data(),
                          out.V.data(), PPC_HOST));
    return out;
}

SvdResult svd(const Matrix& A) {  // matrix_kernels.cpp:29-37
    if (A.rows() < 1 || A.cols() < 1) throw shape_error("svd: empty matrix");
    return truncated_svd(A, std::min(A.rows(), A.cols()));
}

Matrix orthonormalize(const Matrix& A) {
    Matrix Q(A.rows(), A.cols());
    check(ppc_orthonormalize(A.data(), A.rows(), A.cols(), Q.data()));
    return Q;
}

Matrix orthonormal_complement(const Matrix& Q) {  // matrix_kernels.cpp:80-91
    const Index n = Q.rows(), p = Q.cols();
    if (p > n) throw argument_error("orthonormal_complement: more columns than rows");
    if (p == n) return Matrix(n, 0);
    const Matrix P = Matrix::Identity(n, n) - Q * Q.transpose();
    return svd(P).U.leftCols(n - p);
}

Index numerical_rank(const Vector& s, double tol_rel) {  // matrix_kernels.cpp:93-101
    if (s.size() == 0) return 0;
    const double cutoff = tol_rel * s(0);
    Index r = 0;
    while (r < s.size() && s(r) > cutoff) ++r;
    return r;
}

// ---------------------------------------------------------------- transforms
namespace {
Transform built(Matrix Q, TransformKind kind) {
    Transform T;
    T.Q = std::move(Q);
    T.kind = kind;
    return T;
}
}  // namespace

Transform identity_transform(Index n3, Index p) {
    Matrix Q(n3 > 0 ? n3 : 0, p > 0 ? p : 0);
    check(ppc_identity_q(n3, p, Q.data()));
    return built(std::move(Q), TransformKind::Identity);
}

Transform random_orthogonal_transform(Index n3, Index p, std::uint64_t seed) {
    Matrix Q(n3 > 0 ? n3 : 0, p > 0 ? p : 0);
    check(ppc_random_orthogonal_q(n3, p, seed, Q.data()));
    Transform T = built(std::move(Q), TransformKind::RandomOrthogonal);
    T.seed = seed;
    return T;
}

Transform dct_transform(Index n3, Index p) {
    Matrix Q(n3 > 0 ? n3 : 0, p > 0 ? p : 0);
    check(ppc_dct_q(n3, p, Q.data()));
    return built(std::move(Q), TransformKind::Dct);
}

Transform haar_transform(Index n3, Index p) {
    Matrix Q(n3 > 0 ? n3 : 0, p > 0 ? p : 0);
    check(ppc_haar_q(n3, p, Q.data()));
    return built(std::move(Q), TransformKind::Haar);
}

Transform data_dependent_transform(const Tensor3& A, Index p) {  // transforms.cpp:97-115
    Matrix Q(A.n3(), p > 0 ? p : 0);
    int completed = 0;
    check(ppc_data_dependent_q(A.data(), A.n1(), A.n2(), A.n3(), p, Q.data(), nullptr, &completed,
                               PPC_HOST));
    Transform T = built(std::move(Q), TransformKind::DataDependent);
    T.completed_basis = completed != 0;
    return T;
}

Transform custom_transform(Matrix Q, double scale) {  // transforms.cpp:100-111
    check(ppc_check_stiefel(Q.data(), Q.rows(), Q.cols()));
    if (scale == 0.0) throw argument_error("custom_transform: scale must be nonzero");
    Transform T = built(std::move(Q), TransformKind::Custom);
    T.scale = scale;
    return T;
}

Matrix complement_basis(const Transform& T) {  // transforms.cpp:117-162
    const Index n3 = T.n3(), p = T.p();
    if (p == n3) return Matrix(n3, 0);
    Matrix F(n3, n3);
    switch (T.kind) {
        case TransformKind::Identity: check(ppc_identity_q(n3, n3, F.data())); return F.rightCols(n3 - p);
        case TransformKind::Haar: check(ppc_haar_q(n3, n3, F.data())); return F.rightCols(n3 - p);
        case TransformKind::Dct: check(ppc_dct_q(n3, n3, F.data())); return F.rightCols(n3 - p);
        case TransformKind::RandomOrthogonal:
            if (T.seed) {
                check(ppc_random_orthogonal_q(n3, n3, *T.seed, F.data()));
                return F.rightCols(n3 - p);
            }
            break;
        default: break;
    }
    return orthonormal_complement(T.Q);
}

double projection_error(const Tensor3& A, const Transform& T) {  // transforms.cpp:164-174
    if (T.n3() != A.n3())
        throw shape_error("projection_error: transform rows " + std::to_string(T.n3()) +
                          " != tensor n3 " + std::to_string(A.n3()));
    double err = 0.0;
    check(ppc_projection_error(A.data(), A.n1(), A.n2(), A.n3(), T.Q.data(), T.p(), &err, PPC_HOST));
    return err;
}

// -------------------------------------------------------------- star products
StarContext StarContext::with_complement(Transform T) {
    StarContext ctx(std::move(T));
    ctx.complement = complement_basis(ctx.transform);
    return ctx;
}

Tensor3 star_m_product(const Tensor3& A, const Tensor3& B, const Matrix& M) {  // star_products.cpp:38-49
    if (M.rows() != M.cols()) throw shape_error("star_m_product: M must be square");
    if (A.n2() != B.n1())
        throw shape_error("star product: inner extents differ (" + std::to_string(A.n2()) + " vs " +
                          std::to_string(B.n1()) + ")");
    if (A.n3() != M.rows() || B.n3() != M.rows())
        throw shape_error("star product: mode-3 extents must match the transform");
    Tensor3 C(A.n1(), B.n2(), A.n3());
    check(ppc_star_m_product(A.data(), A.n1(), A.n2(), A.n3(), B.data(), B.n2(), M.data(), C.data(), PPC_HOST));
    return C;
}

Tensor3 star_q_product(const Tensor3& A, const Tensor3& B, const StarContext& ctx) {
    const Transform& T = ctx.transform;  // star_products.cpp:13-20
    if (A.n2() != B.n1())
        throw shape_error("star product: inner extents differ (" + std::to_string(A.n2()) + " vs " +
                          std::to_string(B.n1()) + ")");
    if (A.n3() != T.n3() || B.n3() != T.n3())
        throw shape_error("star product: mode-3 extents must match the transform");
    Tensor3 C(A.n1(), B.n2(), A.n3());
    check(ppc_star_q_product(A.data(), A.n1(), A.n2(), A.n3(), B.data(), B.n2(), T.Q.data(), T.p(),
                             T.scale, C.data(), PPC_HOST));
    return C;
}

Tensor3 star_q_identity(Index m, const StarContext& ctx) {  // star_products.cpp:61-72
    if (m < 1) throw argument_error("star_q_identity: m must be positive");
    const Transform& T = ctx.transform;
    Tensor3 Ihat(m, m, T.p());
    for (Index i = 0; i < T.p(); ++i)
        for (Index d = 0; d < m; ++d) Ihat(d, d, i) = 1.0;
    Tensor3 I = mode3_product(Ihat, T.Q);
    if (T.scale != 1.0) I = (1.0 / T.scale) * I;
    return I;
}

Tensor3 star_q_transpose(const Tensor3& A, const StarContext& ctx) {  // star_products.cpp:74-85
    const Transform& T = ctx.transform;
    if (A.n3() != T.n3())
        throw shape_error("star_q_transpose: mode-3 extent " + std::to_string(A.n3()) +
                          " != transform length " + std::to_string(T.n3()));
    Tensor3 Ahat = mode3_product(A, T.Q.transpose());
    Tensor3 Bhat(A.n2(), A.n1(), T.p());
    for (Index i = 0; i < T.p(); ++i) Bhat.set_slice(i, Ahat.slice(i).transpose());
    return mode3_product(Bhat, T.Q);
}

// ------------------------------------------------------------- decompositions
namespace {
void check_transform_match(const Tensor3& A, const Transform& T, const char* who) {
    if (T.n3() != A.n3())
        throw shape_error(std::string(who) + ": transform length " + std::to_string(T.n3()) +
                          " != tensor n3 " + std::to_string(A.n3()));
}
void check_spatial_rank(Index n1, Index n2, Index k, const char* who) {
    const Index cap = std::min(n1, n2);
    if (k < 1 || k > cap)
        throw argument_error(std::string(who) + ": k=" + std::to_string(k) + " outside [1," +
                             std::to_string(cap) + "]");
}
struct Stacks {
    std::vector<double> U, S, V;
};
Stacks pack(const TsvdqFactors& F) {
    const Index p = F.transform.p(), k = F.k;
    if (static_cast<Index>(F.Uhat.size()) != p || static_cast<Index>(F.Vhat.size()) != p ||
        static_cast<Index>(F.shat.size()) != p)
        throw shape_error("tsvdq factors: stack length differs from the transform width");
    Stacks s;
    s.U.resize(static_cast<std::size_t>(F.n1 * k * p));
    s.S.resize(static_cast<std::size_t>(k * p));
    s.V.resize(static_cast<std::size_t>(F.n2 * k * p));
    for (Index i = 0; i < p; ++i) {
        const auto ui = static_cast<std::size_t>(i);
        std::copy(F.Uhat[ui].data(), F.Uhat[ui].data() + F.n1 * k, s.U.data() + i * F.n1 * k);
        std::copy(F.shat[ui].data(), F.shat[ui].data() + k, s.S.data() + i * k);
        std::copy(F.Vhat[ui].data(), F.Vhat[ui].data() + F.n2 * k, s.V.data() + i * F.n2 * k);
    }
    return s;
}
}  // namespace

TsvdqFactors tsvdq(const Tensor3& A, const Transform& T, Index k) {  // decompositions.cpp:62-83
    check_transform_match(A, T, "tsvdq");
    check_spatial_rank(A.n1(), A.n2(), k, "tsvdq");
    const Index p = T.p(), n1 = A.n1(), n2 = A.n2();
    std::vector<double> U(static_cast<std::size_t>(n1 * k * p)), S(static_cast<std::size_t>(k * p)),
        V(static_cast<std::size_t>(n2 * k * p));
    check(ppc_tsvdq(A.data(), n1, n2, A.n3(), T.Q.data(), p, k, U.data(), S.data(), V.data(), PPC_HOST));
    TsvdqFactors F;
    F.transform = T;
    F.k = k;
    F.n1 = n1;
    F.n2 = n2;
    for (Index i = 0; i < p; ++i) {
        Matrix u(n1, k), v(n2, k);
        Vector s(k);
        std::copy(U.data() + i * n1 * k, U.data() + (i + 1) * n1 * k, u.data());
        std::copy(V.data() + i * n2 * k, V.data() + (i + 1) * n2 * k, v.data());
        std::copy(S.data() + i * k, S.data() + (i + 1) * k, s.data());
        F.Uhat.push_back(std::move(u));
        F.shat.push_back(std::move(s));
        F.Vhat.push_back(std::move(v));
    }
    return F;
}

Tensor3 tsvdq_reconstruct(const TsvdqFactors& F) {  // decompositions.cpp:85-94
    const Stacks s = pack(F);
    Tensor3 out(F.n1, F.n2, F.transform.n3());
    check(ppc_tsvdq_reconstruct(s.U.data(), s.S.data(), s.V.data(), F.transform.Q.data(), F.n1, F.n2,
                                F.transform.n3(), F.transform.p(), F.k, out.data(), PPC_HOST));
    return out;
}

ApproxError tsvdq_error(const Tensor3& A, const TsvdqFactors& F) {  // decompositions.cpp:96-103
    check_transform_match(A, F.transform, "tsvdq_error");
    const Stacks s = pack(F);
    ApproxError e;
    check(ppc_tsvdq_error(A.data(), A.n1(), A.n2(), A.n3(), s.U.data(), s.S.data(), s.V.data(),
                          F.transform.Q.data(), F.transform.p(), F.k, &e.total, &e.eckart_young,
                          &e.projection, PPC_HOST));
    return e;
}

Index TsvdqIIFactors::implicit_rank() const {  // decompositions.cpp:116-118
    Index acc = 0;
    for (Index r : multirank) acc += r;
    return acc;
}

TsvdqIIFactors tsvdq2(const Tensor3& A, const Transform& T, double gamma) {  // decompositions.cpp:120-190
    check_transform_match(A, T, "tsvdq2");
    const Index p = T.p(), n1 = A.n1(), n2 = A.n2(), r = std::min(n1, n2);
    std::vector<double> U(static_cast<std::size_t>(n1 * r * p)), S(static_cast<std::size_t>(r * p)),
        V(static_cast<std::size_t>(n2 * r * p));
    std::vector<int64_t> mr(static_cast<std::size_t>(p));
    check(ppc_tsvdq2(A.data(), n1, n2, A.n3(), T.Q.data(), p, gamma, U.data(), S.data(), V.data(),
                     mr.data(), PPC_HOST));
    TsvdqIIFactors F;
    F.gamma = gamma;
    F.transform = T;
    F.n1 = n1;
    F.n2 = n2;
    for (Index i = 0; i < p; ++i) {
        const Index rho = mr[static_cast<std::size_t>(i)];
        F.multirank.push_back(rho);
        Matrix u(n1, rho), v(n2, rho);
        Vector s(rho);
        std::copy(U.data() + i * n1 * r, U.data() + i * n1 * r + n1 * rho, u.data());
        std::copy(V.data() + i * n2 * r, V.data() + i * n2 * r + n2 * rho, v.data());
        std::copy(S.data() + i * r, S.data() + i * r + rho, s.data());
        F.Uhat.push_back(std::move(u));
        F.shat.push_back(std::move(s));
        F.Vhat.push_back(std::move(v));
    }
    return F;
}

namespace {
// Ragged factors -> the padded stacks of ppc_tsvdq2_* (r = min(n1,n2) columns per slice).
Stacks pack2(const TsvdqIIFactors& F, std::vector<int64_t>& mr) {
    const Index p = F.transform.p(), r = std::min(F.n1, F.n2);
    if (static_cast<Index>(F.Uhat.size()) != p || static_cast<Index>(F.Vhat.size()) != p ||
        static_cast<Index>(F.shat.size()) != p || static_cast<Index>(F.multirank.size()) != p)
        throw shape_error("tsvdq2 factors: stack length differs from the transform width");
    Stacks s;
    s.U.assign(static_cast<std::size_t>(F.n1 * r * p), 0.0);
    s.S.assign(static_cast<std::size_t>(r * p), 0.0);
    s.V.assign(static_cast<std::size_t>(F.n2 * r * p), 0.0);
    mr.assign(F.multirank.begin(), F.multirank.end());
    for (Index i = 0; i < p; ++i) {
        const auto ui = static_cast<std::size_t>(i);
        const Index rho = F.multirank[ui];
        if (rho < 0 || rho > r || F.Uhat[ui].cols() != rho || F.Vhat[ui].cols() != rho ||
            F.shat[ui].size() != rho)
            throw shape_error("tsvdq2 factors: slice " + std::to_string(i) + " disagrees with its multirank");
        std::copy(F.Uhat[ui].data(), F.Uhat[ui].data() + F.n1 * rho, s.U.data() + i * F.n1 * r);
        std::copy(F.shat[ui].data(), F.shat[ui].data() + rho, s.S.data() + i * r);
        std::copy(F.Vhat[ui].data(), F.Vhat[ui].data() + F.n2 * rho, s.V.data() + i * F.n2 * r);
    }
    return s;
}
}  // namespace

Tensor3 tsvdq2_reconstruct(const TsvdqIIFactors& F) {  // decompositions.cpp:192-201
    std::vector<int64_t> mr;
    const Stacks s = pack2(F, mr);
    Tensor3 out(F.n1, F.n2, F.transform.n3());
    check(ppc_tsvdq2_reconstruct(s.U.data(), s.S.data(), s.V.data(), F.transform.Q.data(), F.n1, F.n2,
                                 F.transform.n3(), F.transform.p(), mr.data(), out.data(), PPC_HOST));
    return out;
}

ApproxError tsvdq2_error(const Tensor3& A, const TsvdqIIFactors& F) {  // decompositions.cpp:203-209
    check_transform_match(A, F.transform, "tsvdq2_error");
    std::vector<int64_t> mr;
    const Stacks s = pack2(F, mr);
    ApproxError e;
    check(ppc_tsvdq2_error(A.data(), A.n1(), A.n2(), A.n3(), s.U.data(), s.S.data(), s.V.data(),
                           F.transform.Q.data(), F.transform.p(), mr.data(), &e.total, &e.eckart_young,
                           &e.projection, PPC_HOST));
    return e;
}

HosvdFactors hosvd(const Tensor3& A, Index k1, Index k2, Index k3) {  // decompositions.cpp:211-236
    if (k1 < 1 || k1 > A.n1() || k2 < 1 || k2 > A.n2() || k3 < 1 || k3 > A.n3())
        throw argument_error("hosvd: multirank (" + std::to_string(k1) + "," + std::to_string(k2) + "," +
                             std::to_string(k3) + ") outside the tensor extents");
    HosvdFactors F{Tensor3(k1, k2, k3), Matrix(A.n1(), k1), Matrix(A.n2(), k2), Matrix(A.n3(), k3)};
    check(ppc_hosvd(A.data(), A.n1(), A.n2(), A.n3(), k1, k2, k3, F.core.data(), F.U1.data(), F.U2.data(),
                    F.U3.data(), PPC_HOST));
    return F;
}

Tensor3 hosvd_reconstruct(const HosvdFactors& F) {  // decompositions.cpp:238-242
    Tensor3 out(F.U1.rows(), F.U2.rows(), F.U3.rows());
    check(ppc_hosvd_reconstruct(F.core.data(), F.core.n1(), F.core.n2(), F.core.n3(), F.U1.data(), F.U1.rows(),
                                F.U2.data(), F.U2.rows(), F.U3.data(), F.U3.rows(), out.data(), PPC_HOST));
    return out;
}

MatrixSvdBaseline matrix_svd_baseline(const Tensor3& A, Index k) {  // decompositions.cpp:244-255
    const Index cap = std::min(A.n1() * A.n3(), A.n2());
    if (k < 1 || k > cap)
        throw argument_error("matrix_svd_baseline: k=" + std::to_string(k) + " outside [1," +
                             std::to_string(cap) + "]");
    MatrixSvdBaseline out;
    out.factors.U = Matrix(A.n1() * A.n3(), k);
    out.factors.s = Vector(k);
    out.factors.V = Matrix(A.n2(), k);
    check(ppc_matrix_svd_baseline(A.data(), A.n1(), A.n2(), A.n3(), k, out.factors.U.data(),
                                  out.factors.s.data(), out.factors.V.data(), &out.error, PPC_HOST));
    return out;
}

Index star_q_rank(const Tensor3& A, const Transform& T, double tol_rel) {  // decompositions.cpp:105-114
    check_transform_match(A, T, "star_q_rank");
    const Index r = std::min(A.n1(), A.n2()), p = T.p();
    Tensor3 Ahat = mode3_product(A, T.Q.transpose());
    std::vector<double> U(static_cast<std::size_t>(A.n1() * r * p)), S(static_cast<std::size_t>(r * p)),
        V(static_cast<std::size_t>(A.n2() * r * p));
    check(ppc_svd_batched(Ahat.data(), A.n1(), A.n2(), p, r, U.data(), S.data(), V.data(), PPC_HOST));
    Index rank = 0;
    for (Index i = 0; i < p; ++i) {
        Vector s(r);
        std::copy(S.data() + i * r, S.data() + (i + 1) * r, s.data());
        rank = std::max(rank, numerical_rank(s, tol_rel));
    }
    return rank;
}

// --------------------------------------------------------------------- metrics
double relative_error(const Tensor3& A, const Tensor3& Ahat) {  // metrics.cpp:21-28
    if (!A.same_shape(Ahat)) throw shape_error("relative_error: shapes differ");
    double re = 0.0;
    check(ppc_relative_error(A.data(), Ahat.data(), A.size(), &re, PPC_HOST));
    return re;
}

double tsvdq_relative_error(const Tensor3& A, const TsvdqFactors& F) {
    check_transform_match(A, F.transform, "tsvdq_relative_error");
    const Stacks s = pack(F);
    double re = 0.0;
    check(ppc_tsvdq_relative_error(A.data(), A.n1(), A.n2(), A.n3(), s.U.data(), s.S.data(),
                                   s.V.data(), F.transform.Q.data(), F.transform.p(), F.k, &re,
                                   PPC_HOST));
    return re;
}

// --------------------------------------------------------------------- PT3 I/O
void write_pt3(const std::filesystem::path& path, const Tensor3& A) {  // io.cpp:52-70
    check(ppc_pt3_write(path.string().c_str(), A.data(), A.n1(), A.n2(), A.n3(), PPC_HOST));
}

Tensor3 read_pt3(const std::filesystem::path& path) {  // io.cpp:72-112
    int64_t n1 = 0, n2 = 0, n3 = 0;
    check(ppc_pt3_info(path.string().c_str(), &n1, &n2, &n3));
    Tensor3 A(n1, n2, n3);
    check(ppc_pt3_read(path.string().c_str(), A.data(), A.size(), PPC_HOST));
    return A;
}

void write_pt3_matrix(const std::filesystem::path& path, const Matrix& M) {  // io.cpp:114-118
    Tensor3 A(M.rows(), M.cols(), 1);
    A.set_slice(0, M);
    write_pt3(path, A);
}

Matrix read_pt3_matrix(const std::filesystem::path& path) {  // io.cpp:120-126
    Tensor3 A = read_pt3(path);
    if (A.n3() != 1)
        throw format_error(path.string() + ": expected a matrix (n3 = 1), got n3 = " + std::to_string(A.n3()));
    return A.slice(0);
}

// ------------------------------------------------------------ engine controls
namespace engine {
void set_fp64_only(bool on) { check(ppc_set_ozaki(on ? 0 : 1)); }
bool fp64_only() { return ppc_get_ozaki() == 0; }
}  // namespace engine

// ---- parallel.hpp (parallel.cpp:13-57) ------------------------------------
int max_threads() {
    const unsigned hc = std::thread::hardware_concurrency();
    int cap = hc == 0 ? 1 : static_cast<int>(hc);
    if (const char* e = std::getenv("PROJPROD_THREADS"); e && *e) {
        char* end = nullptr;
        const long v = std::strtol(e, &end, 10);
        if (end != e) cap = std::min<long>(cap, std::max<long>(v, 1));  // parsed: clamp to >= 1
    }
    return cap;
}

void parallel_for(std::ptrdiff_t n, const std::function<void(std::ptrdiff_t)>& fn) {
    if (n <= 0) return;
    const std::ptrdiff_t workers = std::min<std::ptrdiff_t>(max_threads(), n);
    const std::ptrdiff_t span = (n + workers - 1) / workers;  // contiguous range per worker
    std::exception_ptr failed;
    std::mutex guard;
    auto run = [&](std::ptrdiff_t lo) {
        try {
            for (std::ptrdiff_t i = lo, hi = std::min(n, lo + span); i < hi; ++i) fn(i);
        } catch (...) {
            std::lock_guard<std::mutex> lk(guard);
            if (!failed) failed = std::current_exception();
        }
    };
    std::vector<std::thread> pool;
    for (std::ptrdiff_t lo = span; lo < n; lo += span) pool.emplace_back(run, lo);
    run(0);  // the first range runs on the calling thread
    for (std::thread& t : pool) t.join();
    if (failed) std::rethrow_exception(failed);
}

}  // namespace projprod
