// Small memory-bound kernels of the engine (deterministic reductions,
// per-column scaling, transposes). All reductions use a fixed grid and a
// fixed summation order, so results are bitwise reproducible run to run and
// independent of the launching device count (verify.cpp:452-455).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace ppc {

constexpr int kReduceBlocks = 1024;  // fixed: reduction order is part of the result
constexpr int kReduceThreads = 256;

// partials[2*b] = sum (a-b)^2, partials[2*b+1] = sum a^2 over block b's
// fixed element subset (b == nullptr: both sums are sum a^2).
void launch_sumsq_partials(const double* a, const double* b, int64_t count, double* partials,
                           cudaStream_t s);
// out[0..1] = fixed-order sums of the pairs in partials[0..2n).
void launch_reduce_pairs(const double* partials, int64_t n, double* out, cudaStream_t s);
// {sum (X - C B)^2, sum X^2} per CTA for a tall product with K <= 32:
// C (M x K, lda), B(k, n) = Bq[n + k * ldb], X (M x Nn, ldx); 2 doubles per
// CTA into partials (smallk_residual_ctas of them), summed by launch_reduce_pairs.
int64_t smallk_residual_ctas(int64_t M, int64_t Nn);
void launch_smallk_residual(const double* Cm, int64_t lda, const double* Bq, int64_t ldb, const double* X,
                            int64_t ldx, int64_t M, int64_t Nn, int64_t K, double* partials, cudaStream_t s);
// out(:, j, b) = U(:, j, b) * S(j, b) for a stack of `batch` rows x k blocks.
void launch_scale_columns(const double* U, const double* S, double* out, int64_t rows,
                          int64_t k, int64_t batch, cudaStream_t s);
// out(:, j, b) = U(:, j, b) * S(j, b) for j < k, where U / S carry kmax
// columns per block (leading-k prefix of a wider factor stack).
void launch_scale_columns_strided(const double* U, const double* S, double* out, int64_t rows, int64_t k,
                                  int64_t kmax, int64_t batch, cudaStream_t s);
// X(:, j, b) = 0 for rank[b] <= j < r: the tail of each block of a padded
// (rows, r, batch) factor stack (rank is a device array of batch entries).
void launch_truncate_columns(double* X, int64_t rows, int64_t r, int64_t batch, const int64_t* rank,
                             cudaStream_t s);
// out(j, i, b) = in(i, j, b) for `batch` rows x cols blocks.
void launch_transpose(const double* in, double* out, int64_t rows, int64_t cols, int64_t batch,
                      cudaStream_t s);
// y = alpha * x
void launch_scale(double* x, int64_t n, double alpha, cudaStream_t s);
// non-finite detector: *flag = 1 if any entry of x is NaN/Inf.
void launch_nonfinite(const double* x, int64_t n, int* flag, cudaStream_t s);

}  // namespace ppc
