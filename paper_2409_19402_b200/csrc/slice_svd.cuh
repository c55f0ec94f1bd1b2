// Facewise SVD / Gram / eigensolver internals (see slice_svd.cu, subspace.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace ppc {

// Problems with min dimension <= this go to the one-CTA Jacobi kernel; larger
// ones to the Gram + Chebyshev-filtered subspace iteration + Rayleigh-Ritz
// polish path (subspace.cu).
constexpr int64_t kSubspaceMinN = 160;

struct GramPlan {
    int64_t chunks = 1;  // power of two
    int64_t chunk = 0;   // rows per chunk (multiple of 16)
};
GramPlan gram_plan(int64_t N, int64_t n3);
// Per-chunk partial Grams of the rows of T (ldT >= rows): parts[c] (n3 x n3).
void gram_partials(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk,
                   int64_t chunks, double* parts, cudaStream_t s, int kshift = 0);
// Fixed pairwise tree over nparts arrays of `elems` doubles; result in parts[0].
void tree_reduce(double* parts, int64_t nparts, int64_t elems, cudaStream_t s);

void subspace_eig_top(const double* G, int64_t n, int64_t batch, int64_t p, double* Q,
                      double* lambda, cudaStream_t s, bool vectors_for_reconstruction);
// Direct top-p eigensolver for one symmetric n x n matrix (tridiag_eig.cu):
// Householder tridiagonalization, bisection, inverse iteration, back-transform.
bool tridiag_eig_eligible(int64_t n, int64_t p, int64_t batch = 1);
// eligible and expected faster than subspace iteration (one cluster per
// matrix, or the whole batch in one wave)
bool tridiag_eig_preferred(int64_t n, int64_t p, int64_t batch);
void tridiag_eig_top(const double* G, int64_t n, int64_t p, double* Q, double* lambda, cudaStream_t s);
// `batch` matrices G + b * strideG: Q (n, p, batch), lambda (p, batch), descending.
void tridiag_eig_top_batched(const double* G, int64_t n, int64_t strideG, int64_t batch, int64_t p, double* Q,
                             double* lambda, cudaStream_t s);
// The direct eigensolve of one matrix in three steps, for the multi-GPU
// driver: the tridiagonalization (replicated), the eigenvalues / inverse
// iteration vectors of an index range (sharded), then the orthonormalization
// of all p vectors (replicated) and the back-transformation of a column range
// (sharded). Every piece gives the bits tridiag_eig_top gives.
struct EigSplit {
    int64_t n, p;
    DeviceBuffer V, tau, d, e, lam, bnd;
    EigSplit(const double* G, int64_t n, int64_t p, cudaStream_t s);
    void vectors(int64_t j0, int64_t j1, double* Z, cudaStream_t s);                     // Z: n x (j1 - j0)
    void finish(double* Zall, int64_t j0, int64_t j1, double* Q, cudaStream_t s);        // Zall: n x p (modified)
};
// Z (r x k per block, column-major, `batch` blocks of r*k) <- orthonormal columns,
// shifted CholQR3 in column order (k <= 160).
void cholqr_inplace(double* Z, int64_t r, int64_t k, cudaStream_t s, int64_t batch = 1);
void slice_tail_energy(const double* A, int64_t m, int64_t n, int64_t stride, int64_t batch,
                       int64_t k, const double* U, const double* S, const double* V, double* tail2,
                       cudaStream_t s);
// Block one-sided Jacobi SVD (block_jacobi.cu) for large slices that keep
// k > r/2 triplets (tsvdq2: k = r): C = min(m, n) in [64, 8192].
bool block_jacobi_eligible(int64_t m, int64_t n, int64_t k);
void block_jacobi_svd(const double* A, int64_t m, int64_t n, int64_t strideA, int64_t batch, int64_t k, double* U,
                      double* S, double* V, double* tail2, cudaStream_t s);
// finite_who (nullable): also check the input for NaN/Inf (PPC_NUMERIC
// "<who>: input has non-finite entries"), inside the slice-Gram split when it
// runs on the INT8 path (returns true then), else not at all (returns false).
bool subspace_svd(const double* A, int64_t m, int64_t n, int64_t stride, int64_t batch, int64_t k,
                  double* U, double* S, double* V, double* tail2, cudaStream_t s, const char* finite_who = nullptr);

}  // namespace ppc
