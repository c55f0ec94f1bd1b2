// Device-level building blocks of the hot path (device pointers, one stream).
// The C-ABI (api.cu) stages host data and calls these; the multi-GPU driver
// composes them per shard.
#pragma once

#include <array>
#include <cstdint>

#include <cuda_runtime.h>

#include "internal.h"

namespace ppc {

// out (N x q) = alpha * T (N x n3) * op(M):  trans_m=false: M is q x n3 (M^T);
// trans_m=true: M is n3 x q (the basis Q itself).       [tensor.cpp:139-147]
void mode3(const double* T, int64_t N, int64_t n3, const double* M, int64_t q, bool trans_m,
           double* out, double alpha, cudaStream_t s);
// The star product's inverse transform C (N x n3) = scale Ch Q^T: the INT8
// row-split kernel (ozaki_star_inverse) where eligible, else mode3 on DMMA.
void star_inverse(const double* Ch, int64_t N, int64_t p, const double* Q, int64_t n3, double scale, double* C,
                  cudaStream_t s);
// C(:,:,i) = A(:,:,i) B(:,:,i), i < p                     [tensor.cpp:149-156]
void facewise(const double* A, int64_t n1, int64_t m, int64_t p, const double* B, int64_t n2,
              double* C, cudaStream_t s);
// The transform-domain facewise product with a strided output (slice i of C
// at C + i*strideC, leading dimension ldc): on the INT8 tensor cores where
// the shapes and the operands' dynamic range allow (as star_q), else FP64
// DMMA. A (n1 x m x p) and B (m x n2 x p) are contiguous slice stacks. Used
// by the row-sharded multi-GPU star-Q, whose C rows are a strided view.
void facewise_auto(const double* A, int64_t n1, int64_t m, int64_t p, const double* B, int64_t n2, double* C,
                   int64_t ldc, int64_t strideC, cudaStream_t s);
// star_products.cpp:51-59
void star_q(const double* A, int64_t n1, int64_t m, int64_t n3, const double* B, int64_t n2,
            const double* Q, int64_t p, double scale, double* C, cudaStream_t s);
// star_q on HOST buffers, pipelined in 2-D tiles: A's row blocks and B's
// lateral blocks stream up alternately, each is transformed as it lands, and
// every tile of C the arrivals complete is computed and sent down at once
// (separate H2D / D2H streams: PCIe runs both directions from the second block
// on). Bitwise equal to star_q on device copies (engine.cu for the argument).
void star_q_host(const double* hA, int64_t n1, int64_t m, int64_t n3, const double* hB, int64_t n2,
                 const double* hQ, int64_t p, double scale, double* hC, cudaStream_t s);
// host sums[0] = sum (a-b)^2 (or a^2 when b == nullptr), sums[1] = sum a^2.
void sumsq(const double* a, const double* b, int64_t count, double sums[2], cudaStream_t s);
// {||T - T Q Q^T||^2, ||T||^2}; coeff (N x p) may be supplied if already known.
std::array<double, 2> projection_residual(const double* T, int64_t N, int64_t n3, const double* Q,
                                          int64_t p, const double* coeff, cudaStream_t s);
// numeric_error if any entry is non-finite (matrix_kernels.cpp:32).
void require_finite(const double* x, int64_t n, const char* who, cudaStream_t s);

// Batched thin SVD (leading k triplets) of `batch` m x n blocks at `stride`.
// tail2 (device, nullable, length batch): sum_{j>=k} s_j^2 per block.
// finite_who (nullable): check the (contiguous) input for NaN/Inf first, as
// the reference's SVD does (matrix_kernels.cpp:32): PPC_NUMERIC "<who>: input
// has non-finite entries" (inside the INT8 slice-Gram split when it runs).
void slice_svd(const double* A, int64_t m, int64_t n, int64_t stride, int64_t batch, int64_t k,
               double* U, double* S, double* V, double* tail2, cudaStream_t s, const char* finite_who = nullptr);

// Deterministic Gram G = T^T T (n3 x n3) over the N rows of T (SYRK).
// nonfinite (nullable device int): when the Gram's own pass over T can also
// detect NaN / Inf it sets *nonfinite on a hit and gram returns true; false
// means T was not checked.
struct OzakiDigits;
// keep (nullable): T's 7-digit split is left there when the INT8 Gram path
// ran on whole 4096-row blocks (reused by the forward transform).
bool gram(const double* T, int64_t N, int64_t n3, double* G, cudaStream_t s, int* nonfinite = nullptr,
          OzakiDigits* keep = nullptr);
// Top-p eigenpairs of a symmetric PSD n x n matrix G: Q (n x p), lambda (p).
// accurate_vectors: lock on the subspace (rank-p truncation) criteria rather
// than on eigenvalues alone.
void sym_eig_top(const double* G, int64_t n, int64_t p, double* Q, double* lambda, cudaStream_t s,
                 bool accurate_vectors = false);
// Partial Grams of nchunks consecutive row chunks (T rows x n3, leading dim ldT).
bool gram_chunks(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk,
                 int64_t nchunks, double* parts, cudaStream_t s, int* nonfinite = nullptr,
                 OzakiDigits* keep = nullptr, int64_t block_base = 0, int64_t total_blocks = 0);
// Eigensolve tail of data_q: Q (sign rule) and sigma from the Gram G.
void eig_to_basis(const double* G, int64_t n3, int64_t p, double* Q, double* sigma, cudaStream_t s,
                  bool accurate_vectors = false);
// Residual sums over a lateral pixel block [j0, j0+nj) (A_blk leading dims n1, ldA).
std::array<double, 2> recon_residual_block(const double* A_blk, int64_t n1, int64_t nj, int64_t n3,
                                           int64_t ldA, const double* U, const double* S,
                                           const double* V, int64_t n2, int64_t j0,
                                           const double* Q, int64_t p, int64_t k, cudaStream_t s);
// transforms.cpp:97-115 on the device. Returns completed_basis.
// check_finite: fail with PPC_NUMERIC on NaN / Inf in T (the svd guard,
// matrix_kernels.cpp:32), folded into the Gram's pass over T where it can be.
// gtrace (device, nullable): trace(G) = ||T||_F^2, from the Gram's diagonal.
bool data_q(const double* T, int64_t N, int64_t n3, int64_t p, double* Q, double* sigma,
            cudaStream_t s, bool check_finite = false, double* gtrace = nullptr, OzakiDigits* keep = nullptr);
// out (device scalar) = trace of the n x n matrix G, fixed summation order.
void gram_trace(const double* G, int64_t n, double* out, cudaStream_t s);
// Finiteness flag for gram / gram_chunks: reset, then test (fails loudly).
struct FiniteFlag {
    int* flag;
    explicit FiniteFlag(cudaStream_t s);
    int* d() { return flag; }
    void check(cudaStream_t s, const char* who);
};

// decompositions.cpp:62-83
// relative_error(A, tsvdq_reconstruct(F)) of the compress chain (metrics.cpp:21-28).
// With Q orthonormal, A - A_k splits into orthogonal parts,
//   ||A - A_k||^2 = (||A||^2 - ||Ahat||^2) + sum_i ||Ahat_i - U_i S_i V_i^T||^2,
// est (device) = {||A||^2 from the Gram trace, the slice residual, ||Ahat||^2}.
// The difference carries ~3e-15 ||A||^2 of rounding, <= 1e-12 relative in RE
// once RE^2 >= 2e-3; below that (or PPC_RE_IDENTITY=0) the residual is
// measured directly against the reconstruction (fused GEMM over A).
double compress_relative_error(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* U,
                               const double* S, const double* V, const double* Q, int64_t p, int64_t k,
                               const double* est, cudaStream_t s);
// out (device, 2 doubles) = {sum_i ||Ahat_i - U_i S_i V_i^T||^2, ||Ahat||^2} over p slices
// Ahat_i (n1 x n2, stride n1*n2): one fused residual GEMM.
void slice_residual_sums(const double* Ah, int64_t n1, int64_t n2, int64_t p, int64_t k, const double* U,
                         const double* S, const double* V, double* out, cudaStream_t s);
// slice_sums (device, nullable, 2 doubles): {sum_i ||Ahat_i - U_i S_i V_i^T||^2, ||Ahat||^2},
// measured directly on the transform-domain slices (fused residual GEMM);
// with a2 (device, ||A||^2) and ||A||^2 - sum s^2 >= 2e-2 ||A||^2 they are
// {0, sum s^2} instead (Eckart-Young through the polish, no pass over Ahat).
// tdig (nullable): A's retained 7-digit Gram split; the forward transform
// then runs on the INT8 tensor cores (ozaki_mode3_forward).
void tsvdq(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* Q, int64_t p,
           int64_t k, double* U, double* S, double* V, cudaStream_t s, double* slice_sums = nullptr,
           const OzakiDigits* tdig = nullptr, const double* a2 = nullptr);
// Chat (n1 x n2 x p) = U diag(S) V^T facewise             [decompositions.cpp:88-92]
// over the leading k columns of factor stacks that carry kstride >= k
// columns per slice (kstride 0 = k).
void core_from_factors(const double* U, const double* S, const double* V, int64_t n1, int64_t n2,
                       int64_t p, int64_t k, double* Chat, cudaStream_t s, int64_t kstride = 0);
// decompositions.cpp:85-94
void reconstruct(const double* U, const double* S, const double* V, const double* Q, int64_t n1,
                 int64_t n2, int64_t n3, int64_t p, int64_t k, double* out, cudaStream_t s,
                 int64_t kstride = 0);
// {||A - recon(F)||^2, ||A||^2} without materializing recon(F).
std::array<double, 2> recon_residual(const double* A, int64_t n1, int64_t n2, int64_t n3,
                                     const double* U, const double* S, const double* V,
                                     const double* Q, int64_t p, int64_t k, cudaStream_t s,
                                     int64_t kstride = 0);
// tools/main.cpp:299-341 sweep, amortized: re[ik + ip*nk] for every (p, k).
void sweep_errors(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* Q, int64_t pmax,
                  int64_t kmax, const int64_t* ps, int64_t np, const int64_t* ks, int64_t nk, double* re,
                  cudaStream_t s);
struct ErrorParts {
    double total, eckart_young, projection;
};
// decompositions.cpp:96-103
ErrorParts tsvdq_error(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* U,
                       const double* S, const double* V, const double* Q, int64_t p, int64_t k,
                       cudaStream_t s);

// decompositions.cpp:120-190 tsvdq2 (energy-truncated multirank). Full slice
// spectra on the device; the global sort and prefix-energy cut over the
// p*r values on the host. Factor stacks padded to r = min(n1,n2) columns
// per slice, zero beyond multirank[i] (host array, p entries).
void tsvdq2(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* Q, int64_t p,
            double gamma, double* U, double* S, double* V, int64_t* multirank, cudaStream_t s);
// The selection alone (decompositions.cpp:131-176): multirank from the full
// spectra s_all (r x p, host, descending per slice).
void tsvdq2_select(const double* s_all, int64_t r, int64_t p, double gamma, int64_t* multirank);
// decompositions.cpp:192-201 on padded factors (only max(multirank) columns used).
void tsvdq2_reconstruct(const double* U, const double* S, const double* V, const double* Q,
                        int64_t n1, int64_t n2, int64_t n3, int64_t p, const int64_t* multirank,
                        double* out, cudaStream_t s);
// decompositions.cpp:203-209
ErrorParts tsvdq2_error(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* U,
                        const double* S, const double* V, const double* Q, int64_t p,
                        const int64_t* multirank, cudaStream_t s);

// SURVEY 8f #4 (baselines.cu)
// star_products.cpp:38-49: [(A x3 M) facewise (B x3 M)] x3 M^{-1}, M n3 x n3.
void star_m(const double* A, int64_t n1, int64_t m, int64_t n3, const double* B, int64_t n2,
            const double* M, double* C, cudaStream_t s);
// tensor.cpp:109-130: A x_m M for m = 1 (out q x n2 x n3) or 2 (out n1 x q x n3),
// M q x n_m column-major; DMMA GEMMs on the buffer as it lies (no unfolding copy).
void mode12_product(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* M, int64_t q,
                    int mode, double* out, cudaStream_t s);
// decompositions.cpp:211-236: core (k1,k2,k3), U1 (n1,k1), U2 (n2,k2), U3 (n3,k3).
void hosvd(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t k1, int64_t k2, int64_t k3,
           double* core, double* U1, double* U2, double* U3, cudaStream_t s);
// decompositions.cpp:238-242
void hosvd_reconstruct(const double* core, int64_t k1, int64_t k2, int64_t k3, const double* U1, int64_t n1,
                       const double* U2, int64_t n2, const double* U3, int64_t n3, double* out,
                       cudaStream_t s);
// decompositions.cpp:244-255: U ((n1 n3) x k), S (k), V (n2 x k); returns the error.
double matrix_svd_baseline(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t k, double* U,
                           double* S, double* V, cudaStream_t s);

}  // namespace ppc
