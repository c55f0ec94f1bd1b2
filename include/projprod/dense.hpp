#pragma once
// Dense column-major matrix / vector types of the projprod C++ API.
//
// The reference defines Matrix/Vector/Index as Eigen::MatrixXd / VectorXd /
// Eigen::Index (proj/include/projprod/tensor.hpp:9-11). Eigen is not part of
// this image, so when <Eigen/Core> is unavailable these are small in-repo
// column-major types with the subset of the Eigen interface the projprod API
// and its callers use (rows/cols/data/operator()/transpose/leftCols/...).
// Define PROJPROD_USE_EIGEN to use Eigen when it is installed.

#if defined(PROJPROD_USE_EIGEN) && __has_include(<Eigen/Core>)
#include <Eigen/Core>
namespace projprod {
using Index = Eigen::Index;
using Matrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
}  // namespace projprod
#else
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <stdexcept>
#include <vector>

namespace projprod {

using Index = std::ptrdiff_t;

class Vector {
public:
    Vector() = default;
    explicit Vector(Index n) : v_(static_cast<std::size_t>(n), 0.0) {}
    Vector(std::initializer_list<double> l) : v_(l) {}
    Index size() const { return static_cast<Index>(v_.size()); }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
    double operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }
    double& operator[](Index i) { return v_[static_cast<std::size_t>(i)]; }
    double operator[](Index i) const { return v_[static_cast<std::size_t>(i)]; }
    Vector head(Index k) const {
        Vector o(k);
        for (Index i = 0; i < k; ++i) o(i) = (*this)(i);
        return o;
    }
    double squaredNorm() const {
        double a = 0;
        for (double x : v_) a += x * x;
        return a;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    static Vector Zero(Index n) { return Vector(n); }

private:
    std::vector<double> v_;
};

class Matrix {
public:
    Matrix() = default;
    Matrix(Index r, Index c) : r_(r), c_(c), v_(static_cast<std::size_t>(r * c), 0.0) {}
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    double& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(i + j * r_)]; }
    double operator()(Index i, Index j) const { return v_[static_cast<std::size_t>(i + j * r_)]; }

    static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
    static Matrix Identity(Index r, Index c) {
        Matrix m(r, c);
        for (Index i = 0; i < (r < c ? r : c); ++i) m(i, i) = 1.0;
        return m;
    }
    Matrix transpose() const {
        Matrix t(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
        return t;
    }
    Matrix middleCols(Index j0, Index k) const {
        if (j0 < 0 || k < 0 || j0 + k > c_) throw std::out_of_range("Matrix::middleCols");
        Matrix o(r_, k);
        for (Index j = 0; j < k; ++j)
            for (Index i = 0; i < r_; ++i) o(i, j) = (*this)(i, j0 + j);
        return o;
    }
    Matrix leftCols(Index k) const { return middleCols(0, k); }
    Matrix rightCols(Index k) const { return middleCols(c_ - k, k); }
    Vector col(Index j) const {
        Vector o(r_);
        for (Index i = 0; i < r_; ++i) o(i) = (*this)(i, j);
        return o;
    }
    double squaredNorm() const {
        double a = 0;
        for (double x : v_) a += x * x;
        return a;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    bool allFinite() const {
        for (double x : v_)
            if (!std::isfinite(x)) return false;
        return true;
    }
    // small host-side helpers for callers and tests (not the engine's path)
    Matrix operator*(const Matrix& b) const {
        if (c_ != b.r_) throw std::invalid_argument("Matrix product: inner dimensions differ");
        Matrix o(r_, b.c_);
        for (Index j = 0; j < b.c_; ++j)
            for (Index k = 0; k < c_; ++k) {
                const double bk = b(k, j);
                for (Index i = 0; i < r_; ++i) o(i, j) += (*this)(i, k) * bk;
            }
        return o;
    }
    Matrix operator-(const Matrix& b) const {
        Matrix o = *this;
        for (std::size_t i = 0; i < v_.size(); ++i) o.v_[i] -= b.v_[i];
        return o;
    }
    Matrix operator+(const Matrix& b) const {
        Matrix o = *this;
        for (std::size_t i = 0; i < v_.size(); ++i) o.v_[i] += b.v_[i];
        return o;
    }

private:
    Index r_ = 0, c_ = 0;
    std::vector<double> v_;
};

inline Matrix operator*(double s, const Matrix& m) {
    Matrix o = m;
    for (Index i = 0; i < o.size(); ++i) o.data()[i] *= s;
    return o;
}

}  // namespace projprod
#endif
