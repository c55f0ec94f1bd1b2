// Batched one-sided Jacobi SVD / small symmetric eigensolver (see jacobi.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace ppc {

size_t jacobi_smem_bytes(int64_t m, int64_t n);
// batch x (m x n) blocks at stride strideA. Leading k triplets (descending):
// U (m,k,batch) [nullable: eigen mode, no sign rule], S (k,batch), V (n,k,batch);
// tail2 (nullable): per-block sum of the squared discarded singular values.
// gtol_rel > 0 (eigen mode only): eigenvalue accuracy gtol_rel * theta_1
// suffices, rotations inside tight clusters below that are skipped.
// sweep_cap > 0 bounds the sweeps (approximate eigenpairs for early
// Rayleigh-Ritz steps of the subspace iteration).
// zmap (device, nullable): launch slot z works on block zmap[z] of the batch
// (batch = number of slots); outputs land at the mapped block.
void jacobi_svd(const double* A, int64_t m, int64_t n, int64_t strideA, int64_t batch, int64_t k,
                double* U, double* S, double* V, double* tail2, cudaStream_t s, double gtol_rel = 0.0,
                int sweep_cap = 0, const int* zmap = nullptr);
// Sign rule of matrix_kernels.cpp:16-25 on `batch` stacks of X (rows x cols):
// the largest-|x| entry (first on ties) of each column made nonnegative; the
// matching column of Y (yrows x cols, nullable) is flipped with it.
void sign_rule(double* X, int64_t rows, int64_t cols, int64_t batch, double* Y, int64_t yrows,
               cudaStream_t s);

}  // namespace ppc
