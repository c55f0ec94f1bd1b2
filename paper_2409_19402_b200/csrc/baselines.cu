// the star-M product and the Tucker / flattened-SVD baselines
// the reference compares the projected SVD against, composed from the hot
// path's own kernels (DMMA mode products and SYRKs, the Gram eigensolver,
// the batched slice SVD and the fused residual GEMM).
#include <algorithm>
#include <cmath>
#include <vector>

#include "dmma_gemm.cuh"
#include "engine.h"
#include "internal.h"
#include "jacobi.cuh"
#include "kernels.cuh"
#include "slice_svd.cuh"

namespace ppc {

namespace {

__global__ void inv_scale_columns_kernel(const double* __restrict__ V, const double* __restrict__ s,
                                         double* __restrict__ out, int64_t rows, int64_t total) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
        out[i] = V[i] / s[i / rows];
}

// G (rows x rows) = X X^T for X rows x K column-major (leading dim rows):
// the Gram of a mode unfolding (symmetric DMMA SYRK, fixed summation order).
void unfolding_gram(const double* X, int64_t rows, int64_t K, double* G, cudaStream_t s) {
    GemmDesc d;
    d.M = rows; d.N = rows; d.K = K; d.symmetric = true;
    d.A = X; d.lda = rows; d.a_kmajor = false;      // A(mm,kk) = X[mm + kk*rows]
    d.B = X; d.ldb = rows; d.b_nmajor = true;       // B(kk,nn) = X[nn + kk*rows]
    d.C = G; d.ldc = rows;
    gemm(d, s);
}

// hosvd_factor (decompositions.cpp:216-227): leading ki left singular vectors
// of the unfolding = top eigenvectors of its Gram, sign rule applied. Beyond
// the unfolding's rank the Gram's null-space eigenvectors complete the basis.
// The factors feed a reconstruction, so the eigensolver locks on subspace
// accuracy, not on eigenvalues alone.
void mode_factor(const double* G, int64_t rows, int64_t ki, double* U, cudaStream_t s) {
    eig_to_basis(G, rows, ki, U, nullptr, s, true);
}

}  // namespace

void star_m(const double* A, int64_t n1, int64_t m, int64_t n3, const double* B, int64_t n2,
            const double* M, double* C, cudaStream_t s) {
    // star_products.cpp:38-49: M^{-1} = V diag(1/s) U^T from the SVD of M,
    // after the numerical-rank gate (numerical_rank, matrix_kernels.cpp:93-101).
    DeviceBuffer u(sizeof(double) * n3 * n3), sv(sizeof(double) * n3), v(sizeof(double) * n3 * n3),
        vs(sizeof(double) * n3 * n3), minv(sizeof(double) * n3 * n3);
    require_finite(M, n3 * n3, "svd", s);
    slice_svd(M, n3, n3, n3 * n3, 1, n3, u.d(), sv.d(), v.d(), nullptr, s);
    std::vector<double> sh(n3);
    PPC_CUDA_CHECK(cudaMemcpyAsync(sh.data(), sv.d(), sizeof(double) * n3, cudaMemcpyDeviceToHost, s));
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    int64_t rank = 0;
    while (rank < n3 && sh[rank] > 1e-12 * sh[0]) ++rank;
    if (rank < n3) fail(PPC_DEGENERATE, "star_m_product: M is numerically singular");
    inv_scale_columns_kernel<<<(unsigned)std::min<int64_t>((n3 * n3 + 255) / 256, 148 * 16), 256, 0, s>>>(
        v.d(), sv.d(), vs.d(), n3, n3 * n3);
    count_launch();
    check_launch("inv_scale_columns");
    {
        GemmDesc d;  // Minv = (V diag(1/s)) U^T
        d.M = n3; d.N = n3; d.K = n3;
        d.A = vs.d(); d.lda = n3;
        d.B = u.d(); d.ldb = n3; d.b_nmajor = true;
        d.C = minv.d(); d.ldc = n3;
        gemm(d, s);
    }
    DeviceBuffer ah(sizeof(double) * n1 * m * n3), bh(sizeof(double) * m * n2 * n3),
        ch(sizeof(double) * n1 * n2 * n3);
    mode3(A, n1 * m, n3, M, n3, false, ah.d(), 1.0, s);   // A x3 M
    mode3(B, m * n2, n3, M, n3, false, bh.d(), 1.0, s);   // B x3 M
    facewise(ah.d(), n1, m, n3, bh.d(), n2, ch.d(), s);
    mode3(ch.d(), n1 * n2, n3, minv.d(), n3, false, C, 1.0, s);  // x3 M^{-1}
}

void mode12_product(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* M, int64_t q,
                     int mode, double* out, cudaStream_t s) {
    GemmDesc d;
    if (mode == 1) {
        // tensor.cpp:112-120: out(:,:,k) = M A(:,:,k); the buffer is the
        // n1 x (n2 n3) mode-1 unfolding, so this is one GEMM
        d.M = q; d.N = n2 * n3; d.K = n1;
        d.A = M; d.lda = q;
        d.B = A; d.ldb = n1;
        d.C = out; d.ldc = q;
    } else {
        // tensor.cpp:121-130: out(:,:,k) = A(:,:,k) M^T, batched over the slices
        d.M = n1; d.N = q; d.K = n2; d.batch = n3;
        d.A = A; d.lda = n1; d.strideA = n1 * n2;
        d.B = M; d.ldb = q; d.strideB = 0; d.b_nmajor = true;  // B(kk,nn) = M[nn + kk*q]
        d.C = out; d.ldc = n1; d.strideC = n1 * q;
    }
    gemm(d, s);
}

void hosvd(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t k1, int64_t k2, int64_t k3,
           double* core, double* U1, double* U2, double* U3, cudaStream_t s) {
    const int64_t N = n1 * n2;
    require_finite(A, N * n3, "svd", s);
    {  // mode 1: the buffer itself is the n1 x (n2 n3) unfolding (tensor.cpp:89-94)
        DeviceBuffer G(sizeof(double) * n1 * n1);
        unfolding_gram(A, n1, n2 * n3, G.d(), s);
        mode_factor(G.d(), n1, k1, U1, s);
    }
    {  // mode 2: slice-wise transposes give the n2 x (n1 n3) unfolding (:95-100)
        DeviceBuffer At(sizeof(double) * N * n3), G(sizeof(double) * n2 * n2);
        launch_transpose(A, At.d(), n1, n2, n3, s);
        unfolding_gram(At.d(), n2, n1 * n3, G.d(), s);
        mode_factor(G.d(), n2, k2, U2, s);
    }
    {  // mode 3: the tube-matrix Gram of the data-driven transform
        DeviceBuffer G(sizeof(double) * n3 * n3);
        gram(A, N, n3, G.d(), s);
        mode_factor(G.d(), n3, k3, U3, s);
    }
    // core = A x1 U1^T x2 U2^T x3 U3^T (decompositions.cpp:231-234, same order)
    DeviceBuffer y1(sizeof(double) * k1 * n2 * n3), y2(sizeof(double) * k1 * k2 * n3);
    {
        GemmDesc d;  // Y1 (k1 x n2 n3) = U1^T X1
        d.M = k1; d.N = n2 * n3; d.K = n1;
        d.A = U1; d.lda = n1; d.a_kmajor = true;
        d.B = A; d.ldb = n1;
        d.C = y1.d(); d.ldc = k1;
        gemm(d, s);
    }
    {
        GemmDesc d;  // per slice: Y2_k (k1 x k2) = Y1_k (k1 x n2) U2 (n2 x k2)
        d.M = k1; d.N = k2; d.K = n2; d.batch = n3;
        d.A = y1.d(); d.lda = k1; d.strideA = k1 * n2;
        d.B = U2; d.ldb = n2; d.strideB = 0;
        d.C = y2.d(); d.ldc = k1; d.strideC = k1 * k2;
        gemm(d, s);
    }
    mode3(y2.d(), k1 * k2, n3, U3, k3, true, core, 1.0, s);
}

void hosvd_reconstruct(const double* core, int64_t k1, int64_t k2, int64_t k3, const double* U1, int64_t n1,
                       const double* U2, int64_t n2, const double* U3, int64_t n3, double* out,
                       cudaStream_t s) {
    // decompositions.cpp:238-242: core x1 U1 x2 U2 x3 U3
    DeviceBuffer z1(sizeof(double) * n1 * k2 * k3), z2(sizeof(double) * n1 * n2 * k3);
    {
        GemmDesc d;  // Z1 (n1 x k2 k3) = U1 core_(1)
        d.M = n1; d.N = k2 * k3; d.K = k1;
        d.A = U1; d.lda = n1;
        d.B = core; d.ldb = k1;
        d.C = z1.d(); d.ldc = n1;
        gemm(d, s);
    }
    {
        GemmDesc d;  // per slice: Z2_k (n1 x n2) = Z1_k (n1 x k2) U2^T
        d.M = n1; d.N = n2; d.K = k2; d.batch = k3;
        d.A = z1.d(); d.lda = n1; d.strideA = n1 * k2;
        d.B = U2; d.ldb = n2; d.strideB = 0; d.b_nmajor = true;
        d.C = z2.d(); d.ldc = n1; d.strideC = n1 * n2;
        gemm(d, s);
    }
    mode3(z2.d(), n1 * n2, k3, U3, n3, false, out, 1.0, s);
}

double matrix_svd_baseline(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t k, double* U,
                           double* S, double* V, cudaStream_t s) {
    // decompositions.cpp:244-255: B = the (n1 n3) x n2 stack of frontal
    // slices. B^T is the mode-2 unfolding, i.e. the slice-wise transpose.
    const int64_t R = n1 * n3;
    require_finite(A, n1 * n2 * n3, "svd", s);
    DeviceBuffer Bt(sizeof(double) * n2 * R);
    launch_transpose(A, Bt.d(), n1, n2, n3, s);
    // B^T = Ut S Vt^T  =>  B = Vt S Ut^T: U = Vt (R x k), V = Ut (n2 x k)
    slice_svd(Bt.d(), n2, R, n2 * R, 1, k, V, S, U, nullptr, s);
    sign_rule(U, R, k, 1, V, n2, s);  // fix_svd_signs on B's U (matrix_kernels.cpp:16-25)
    // error = ||B - U S V^T|| = ||B^T - V S U^T||, measured by the fused residual
    DeviceBuffer vs(sizeof(double) * n2 * k);
    launch_scale_columns(V, S, vs.d(), n2, k, 1, s);
    GemmDesc d;
    d.M = n2; d.N = R; d.K = k;
    d.A = vs.d(); d.lda = n2;
    d.B = U; d.ldb = R; d.b_nmajor = true;
    const int64_t ctas = gemm_residual_ctas(d, Bt.d(), n2, 0);
    DeviceBuffer part(sizeof(double) * 2 * (ctas + 1));
    gemm_residual(d, Bt.d(), n2, 0, part.d(), s);
    double* fin = part.d() + 2 * ctas;
    launch_reduce_pairs(part.d(), ctas, fin, s);
    double sums[2];
    PPC_CUDA_CHECK(cudaMemcpyAsync(sums, fin, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    return std::sqrt(sums[0]);
}

}  // namespace ppc
