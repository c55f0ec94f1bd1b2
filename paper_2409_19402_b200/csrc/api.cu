// C-ABI entry points (include/ppc.h). Each function validates its arguments
// with the reference's checks and messages (thrown before any work starts, as
// in tensor.cpp:140-142, decompositions.cpp:16-28, star_products.cpp:13-20),
// then drives the device kernels on the calling thread's stream.
#include <algorithm>
#include <cmath>
#include <string>
#include <memory>
#include <map>

#include "dmma_gemm.cuh"
#include "internal.h"
#include "jacobi.cuh"
#include "kernels.cuh"
#include "engine.h"
#include "ozaki.h"
#include "slice_svd.cuh"

using namespace ppc;

namespace {

std::string shp(int64_t a, int64_t b, int64_t c) {
    return std::to_string(a) + "x" + std::to_string(b) + "x" + std::to_string(c);
}

void check_tensor(int64_t n1, int64_t n2, int64_t n3) {
    if (n1 < 1 || n2 < 1 || n3 < 1)
        fail(PPC_SHAPE, "tensor extents must be positive, got " + shp(n1, n2, n3));
}

// transforms.cpp:15-20
void check_transform(int64_t n3, int64_t p) {
    if (n3 < 1) fail(PPC_ARGUMENT, "transform: n3 must be positive");
    if (p < 1 || p > n3)
        fail(PPC_ARGUMENT,
             "transform: p=" + std::to_string(p) + " outside [1," + std::to_string(n3) + "]");
}

// decompositions.cpp:23-28
void check_spatial_rank(int64_t n1, int64_t n2, int64_t k, const char* who) {
    const int64_t cap = n1 < n2 ? n1 : n2;
    if (k < 1 || k > cap)
        fail(PPC_ARGUMENT, std::string(who) + ": k=" + std::to_string(k) + " outside [1," +
                               std::to_string(cap) + "]");
}

}  // namespace

namespace {
// Host input: stream A in row-chunk groups on the copy stream into abuf and
// start each group's partial Grams as soon as it lands (the H2D overlaps
// the SYRK); then Q (n3 x p) from the Gram. Same chunks and tree as the
// resident path, so Q is bitwise identical. `tdig` keeps the groups' digit
// split for the forward transform, `trace` receives trace(G).
void host_streamed_q(const double* A, int64_t N, int64_t n3, int64_t p, DeviceBuffer& abuf, double* Qout,
                     double* sigma, double* trace, OzakiDigits* tdig, cudaStream_t s) {
    if (!A) fail(PPC_ARGUMENT, "null input pointer");
    abuf = DeviceBuffer(sizeof(double) * N * n3);
    const GramPlan g = gram_plan(N, n3);
    const int64_t per = std::min<int64_t>(g.chunks, 4);  // chunks per upload group
    DeviceBuffer parts(sizeof(double) * g.chunks * n3 * n3);
    cudaStream_t cs = copy_stream();
    {
        // the staging buffer was allocated on s: order cs after it
        cudaEvent_t ready;
        PPC_CUDA_CHECK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        PPC_CUDA_CHECK(cudaEventRecord(ready, s));
        PPC_CUDA_CHECK(cudaStreamWaitEvent(cs, ready, 0));
        PPC_CUDA_CHECK(cudaEventDestroy(ready));
    }
    FiniteFlag nf(s);
    bool checked = true;  // every slab's Gram pass also checked finiteness (INT8 path)
    // the groups' digits land in one allocation, block c0 * blk_per_chunk on
    const int64_t blk_per_chunk = (g.chunk + 4095) / 4096;
    const bool keep = tdig && g.chunk % 4096 == 0;
    {
        StageTimer tm("gram_syrk", s, (double)N * n3 * n3, 8.0 * N * n3);
        // groups of `per` chunks; the last chunk travels alone, so the
        // Gram work left after the final byte lands is one chunk's
        for (int64_t c0 = 0, take = 0; c0 < g.chunks; c0 += take) {
            take = std::min<int64_t>(per, g.chunks - c0);
            if (take > 1 && c0 + take == g.chunks) --take;
            const int64_t r0 = c0 * g.chunk;
            if (r0 >= N) {  // plan chunks beyond N: zero partials
                PPC_CUDA_CHECK(cudaMemsetAsync(parts.d() + c0 * n3 * n3, 0,
                                               sizeof(double) * (g.chunks - c0) * n3 * n3, s));
                break;
            }
            const int64_t nr = std::min<int64_t>(take * g.chunk, N - r0);
            PPC_CUDA_CHECK(cudaMemcpy2DAsync(abuf.d() + r0, sizeof(double) * N, A + r0, sizeof(double) * N,
                                             sizeof(double) * nr, n3, cudaMemcpyHostToDevice, cs));
            cudaEvent_t ev;
            PPC_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            PPC_CUDA_CHECK(cudaEventRecord(ev, cs));
            PPC_CUDA_CHECK(cudaStreamWaitEvent(s, ev, 0));
            PPC_CUDA_CHECK(cudaEventDestroy(ev));
            checked &= gram_chunks(abuf.d() + r0, N, nr, n3, g.chunk, take,
                                   parts.d() + c0 * n3 * n3, s, nf.d(), keep ? tdig : nullptr,
                                   c0 * blk_per_chunk, g.chunks * blk_per_chunk);
        }
        tree_reduce(parts.d(), g.chunks, n3 * n3, s);
    }
    if (tdig) tdig->uniform = keep && checked && tdig->nd == 7;  // every group on the INT8 path
    if (checked)
        nf.check(s, "svd");
    else
        require_finite(abuf.d(), N * n3, "svd", s);
    if (trace) gram_trace(parts.d(), n3, trace, s);
    eig_to_basis(parts.d(), n3, p, Qout, sigma, s);
}

}  // namespace

extern "C" {

int ppc_mode3_product(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* M,
                      int64_t q, int trans_m, double* out, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        if (q < 1) fail(PPC_SHAPE, "mode3_product: M must have at least one row");
        const int64_t N = n1 * n2;
        cudaStream_t s = stream();
        In a(A, N * n3, loc), m(M, q * n3, loc);
        Out o(out, N * q, loc);
        mode3(a.d, N, n3, m.d, q, trans_m != 0, o.d, 1.0, s);
        o.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_mode_product(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* M,
                     int64_t q, int mode, double* out, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        if (mode < 1 || mode > 3)
            fail(PPC_ARGUMENT, "mode_product: mode must be 1, 2 or 3, got " + std::to_string(mode));
        if (q < 1) fail(PPC_SHAPE, "mode_product: M must have at least one row");
        const int64_t ext = mode == 1 ? n1 : (mode == 2 ? n2 : n3);
        const int64_t count = n1 * n2 * n3 / ext * q;
        cudaStream_t s = stream();
        In a(A, n1 * n2 * n3, loc), m(M, q * ext, loc);
        Out o(out, count, loc);
        if (mode == 3) mode3(a.d, n1 * n2, n3, m.d, q, false, o.d, 1.0, s);
        else mode12_product(a.d, n1, n2, n3, m.d, q, mode, o.d, s);
        o.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_facewise_product(const double* A, int64_t n1, int64_t m, int64_t n3, const double* B,
                         int64_t n2, double* C, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, m, n3);
        check_tensor(m, n2, n3);
        cudaStream_t s = stream();
        In a(A, n1 * m * n3, loc), b(B, m * n2 * n3, loc);
        Out c(C, n1 * n2 * n3, loc);
        facewise(a.d, n1, m, n3, b.d, n2, c.d, s);
        c.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_frobenius_norm(const double* A, int64_t count, double* out, int loc) {
    return guarded([&] {
        validate_loc(loc);
        if (count < 0) fail(PPC_SHAPE, "frobenius_norm: negative count");
        if (!out) fail(PPC_ARGUMENT, "null output");
        cudaStream_t s = stream();
        In a(A, count, loc);
        double sums[2];
        sumsq(a.d, nullptr, count, sums, s);
        *out = std::sqrt(sums[1]);
    });
}

int ppc_relative_error(const double* A, const double* Ahat, int64_t count, double* re, int loc) {
    return guarded([&] {
        validate_loc(loc);
        if (count < 1) fail(PPC_SHAPE, "relative_error: shapes differ");
        if (!re) fail(PPC_ARGUMENT, "null output");
        cudaStream_t s = stream();
        In a(A, count, loc), b(Ahat, count, loc);
        double sums[2];
        sumsq(a.d, b.d, count, sums, s);
        // metrics.cpp:23-27
        if (sums[1] == 0.0) fail(PPC_DEGENERATE, "relative_error: reference tensor is zero");
        *re = std::sqrt(sums[0]) / std::sqrt(sums[1]);
    });
}

int ppc_projection_error(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* Q,
                         int64_t p, double* err, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        check_transform(n3, p);
        if (!err) fail(PPC_ARGUMENT, "null output");
        cudaStream_t s = stream();
        const int64_t N = n1 * n2;
        In a(A, N * n3, loc), q(Q, n3 * p, loc);
        *err = std::sqrt(projection_residual(a.d, N, n3, q.d, p, nullptr, s)[0]);
    });
}

int ppc_star_q_product(const double* A, int64_t n1, int64_t m, int64_t n3, const double* B,
                       int64_t n2, const double* Q, int64_t p, double scale, double* C, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, m, n3);
        check_tensor(m, n2, n3);
        check_transform(n3, p);
        cudaStream_t s = stream();
        if (loc == PPC_HOST) {  // PCIe both ways at once behind the compute
            if (!A || !B || !Q || !C) fail(PPC_ARGUMENT, "null pointer");
            star_q_host(A, n1, m, n3, B, n2, Q, p, scale, C, s);
            PPC_CUDA_CHECK(cudaStreamSynchronize(s));
            return;
        }
        In a(A, n1 * m * n3, loc), b(B, m * n2 * n3, loc), q(Q, n3 * p, loc);
        Out c(C, n1 * n2 * n3, loc);
        star_q(a.d, n1, m, n3, b.d, n2, q.d, p, scale, c.d, s);
        c.finish();
    });
}

int ppc_svd_batched(const double* A, int64_t m, int64_t n, int64_t batch, int64_t k, double* U,
                    double* S, double* V, int loc) {
    return guarded([&] {
        validate_loc(loc);
        if (m < 1 || n < 1) fail(PPC_SHAPE, "svd: empty matrix");
        if (batch < 1) fail(PPC_SHAPE, "svd: batch must be positive");
        const int64_t r = m < n ? m : n;
        if (k < 1 || k > r)
            fail(PPC_ARGUMENT, "truncated_svd: k=" + std::to_string(k) + " outside [1," +
                                   std::to_string(r) + "]");
        cudaStream_t s = stream();
        In a(A, m * n * batch, loc);
        require_finite(a.d, m * n * batch, "svd", s);
        Out u(U, m * k * batch, loc), sv(S, k * batch, loc), v(V, n * k * batch, loc);
        slice_svd(a.d, m, n, m * n, batch, k, u.d, sv.d, v.d, nullptr, s);
        u.finish();
        sv.finish();
        v.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_data_dependent_q(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t p,
                         double* Q, double* sigma, int* completed, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_transform(n3, p);  // transforms.cpp:98
        check_tensor(n1, n2, n3);
        cudaStream_t s = stream();
        const int64_t N = n1 * n2;
        In a(A, N * n3, loc);
        Out q(Q, n3 * p, loc);
        Out sg(sigma, sigma ? p : 0, loc);
        const bool comp = data_q(a.d, N, n3, p, q.d, sigma ? sg.d : nullptr, s, true);
        if (completed) *completed = comp ? 1 : 0;
        q.finish();
        if (sigma) sg.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_tsvdq(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* Q, int64_t p,
              int64_t k, double* U, double* S, double* V, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        check_transform(n3, p);
        check_spatial_rank(n1, n2, k, "tsvdq");
        cudaStream_t s = stream();
        In a(A, n1 * n2 * n3, loc), q(Q, n3 * p, loc);
        Out u(U, n1 * k * p, loc), sv(S, k * p, loc), v(V, n2 * k * p, loc);
        tsvdq(a.d, n1, n2, n3, q.d, p, k, u.d, sv.d, v.d, s);
        u.finish();
        sv.finish();
        v.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_tsvdq_reconstruct(const double* U, const double* S, const double* V, const double* Q,
                          int64_t n1, int64_t n2, int64_t n3, int64_t p, int64_t k, double* out,
                          int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        check_transform(n3, p);
        check_spatial_rank(n1, n2, k, "tsvdq_reconstruct");
        cudaStream_t s = stream();
        In u(U, n1 * k * p, loc), sv(S, k * p, loc), v(V, n2 * k * p, loc), q(Q, n3 * p, loc);
        Out o(out, n1 * n2 * n3, loc);
        reconstruct(u.d, sv.d, v.d, q.d, n1, n2, n3, p, k, o.d, s);
        o.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_tsvdq_error(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* U,
                    const double* S, const double* V, const double* Q, int64_t p, int64_t k,
                    double* total, double* eckart_young, double* projection, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        check_transform(n3, p);  // decompositions.cpp:97 check_transform_match
        check_spatial_rank(n1, n2, k, "tsvdq_error");
        if (!total || !eckart_young || !projection) fail(PPC_ARGUMENT, "null output");
        cudaStream_t s = stream();
        In a(A, n1 * n2 * n3, loc), u(U, n1 * k * p, loc), sv(S, k * p, loc), v(V, n2 * k * p, loc),
            q(Q, n3 * p, loc);
        const ErrorParts e = tsvdq_error(a.d, n1, n2, n3, u.d, sv.d, v.d, q.d, p, k, s);
        *total = e.total;
        *eckart_young = e.eckart_young;
        *projection = e.projection;
    });
}

int ppc_tsvdq_relative_error(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* U,
                             const double* S, const double* V, const double* Q, int64_t p,
                             int64_t k, double* re, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        check_transform(n3, p);
        check_spatial_rank(n1, n2, k, "tsvdq_relative_error");
        if (!re) fail(PPC_ARGUMENT, "null output");
        cudaStream_t s = stream();
        In a(A, n1 * n2 * n3, loc), u(U, n1 * k * p, loc), sv(S, k * p, loc), v(V, n2 * k * p, loc),
            q(Q, n3 * p, loc);
        const auto r = recon_residual(a.d, n1, n2, n3, u.d, sv.d, v.d, q.d, p, k, s);
        if (r[1] == 0.0) fail(PPC_DEGENERATE, "relative_error: reference tensor is zero");
        *re = std::sqrt(r[0]) / std::sqrt(r[1]);
    });
}

namespace {

void check_multirank(const int64_t* multirank, int64_t p, int64_t r, const char* who) {
    if (!multirank) fail(PPC_ARGUMENT, std::string(who) + ": null multirank");
    for (int64_t i = 0; i < p; ++i)
        if (multirank[i] < 0 || multirank[i] > r)
            fail(PPC_BOUNDS, std::string(who) + ": multirank[" + std::to_string(i) + "]=" +
                                 std::to_string(multirank[i]) + " outside [0," + std::to_string(r) + "]");
}

}  // namespace

int ppc_tsvdq2(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* Q, int64_t p,
               double gamma, double* U, double* S, double* V, int64_t* multirank, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        check_transform(n3, p);  // decompositions.cpp:121
        if (!(gamma > 0.0 && gamma <= 1.0))  // :122-124
            fail(PPC_ARGUMENT, "tsvdq2: gamma must lie in (0,1], got " + std::to_string(gamma));
        if (!multirank) fail(PPC_ARGUMENT, "tsvdq2: null multirank");
        const int64_t r = std::min(n1, n2);
        cudaStream_t s = stream();
        In a(A, n1 * n2 * n3, loc), q(Q, n3 * p, loc);
        Out u(U, n1 * r * p, loc), sv(S, r * p, loc), v(V, n2 * r * p, loc);
        tsvdq2(a.d, n1, n2, n3, q.d, p, gamma, u.d, sv.d, v.d, multirank, s);
        u.finish();
        sv.finish();
        v.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_tsvdq2_reconstruct(const double* U, const double* S, const double* V, const double* Q,
                           int64_t n1, int64_t n2, int64_t n3, int64_t p, const int64_t* multirank,
                           double* out, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        check_transform(n3, p);
        const int64_t r = std::min(n1, n2);
        check_multirank(multirank, p, r, "tsvdq2_reconstruct");
        cudaStream_t s = stream();
        In u(U, n1 * r * p, loc), sv(S, r * p, loc), v(V, n2 * r * p, loc), q(Q, n3 * p, loc);
        Out o(out, n1 * n2 * n3, loc);
        tsvdq2_reconstruct(u.d, sv.d, v.d, q.d, n1, n2, n3, p, multirank, o.d, s);
        o.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_tsvdq2_error(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* U,
                     const double* S, const double* V, const double* Q, int64_t p,
                     const int64_t* multirank, double* total, double* eckart_young,
                     double* projection, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        check_transform(n3, p);  // decompositions.cpp:204
        if (!total || !eckart_young || !projection) fail(PPC_ARGUMENT, "null output");
        const int64_t r = std::min(n1, n2);
        check_multirank(multirank, p, r, "tsvdq2_error");
        cudaStream_t s = stream();
        In a(A, n1 * n2 * n3, loc), u(U, n1 * r * p, loc), sv(S, r * p, loc), v(V, n2 * r * p, loc),
            q(Q, n3 * p, loc);
        const ErrorParts e = tsvdq2_error(a.d, n1, n2, n3, u.d, sv.d, v.d, q.d, p, multirank, s);
        *total = e.total;
        *eckart_young = e.eckart_young;
        *projection = e.projection;
    });
}

int ppc_gemm_strided(int64_t M, int64_t N, int64_t K, int64_t batch, double alpha, const double* A,
                     int64_t lda, int64_t strideA, int trans_a, const double* B, int64_t ldb,
                     int64_t strideB, int trans_b, double* C, int64_t ldc, int64_t strideC) {
    return guarded([&] {
        if (M < 0 || N < 0 || K < 0 || batch < 0) fail(PPC_SHAPE, "gemm_strided: negative extent");
        if (!M || !N || !batch) return;
        if (!A || !B || !C) fail(PPC_ARGUMENT, "gemm_strided: null operand");
        if (lda < (trans_a ? K : M) || ldb < (trans_b ? N : K) || ldc < M)
            fail(PPC_ARGUMENT, "gemm_strided: leading dimension too small");
        GemmDesc d;
        d.M = M; d.N = N; d.K = K; d.batch = batch;
        d.A = A; d.lda = lda; d.strideA = strideA; d.a_kmajor = trans_a != 0;
        d.B = B; d.ldb = ldb; d.strideB = strideB; d.b_nmajor = trans_b != 0;
        d.C = C; d.ldc = ldc; d.strideC = strideC;
        d.alpha = alpha;
        if (K == 0) {  // empty sum: C = 0
            for (int64_t b = 0; b < batch; ++b)
                PPC_CUDA_CHECK(cudaMemset2DAsync(C + b * strideC, sizeof(double) * ldc, 0, sizeof(double) * M,
                                                 (size_t)N, stream()));
            return;
        }
        gemm(d, stream());
    });
}

int ppc_facewise_strided(const double* A, int64_t n1, int64_t m, int64_t batch, const double* B, int64_t n2,
                         double* C, int64_t ldc, int64_t strideC) {
    return guarded([&] {
        check_tensor(n1, m, batch);
        require_positive(n2, "n2");
        if (!A || !B || !C) fail(PPC_ARGUMENT, "facewise_strided: null operand");
        if (ldc < n1 || strideC < ldc * n2) fail(PPC_ARGUMENT, "facewise_strided: output strides too small");
        facewise_auto(A, n1, m, batch, B, n2, C, ldc, strideC, stream());
    });
}

int ppc_star_inverse(const double* Ch, int64_t N, int64_t p, const double* Q, int64_t n3, double scale, double* C) {
    return guarded([&] {
        require_positive(N, "N");
        require_positive(p, "p");
        require_positive(n3, "n3");
        if (!Ch || !Q || !C) fail(PPC_ARGUMENT, "star_inverse: null operand");
        star_inverse(Ch, N, p, Q, n3, scale, C, stream());
    });
}

int ppc_reshard_slices(const double* recv, int64_t G, int64_t ps, int64_t nj, int64_t n1, double* out) {
    return guarded([&] {
        if (G < 1 || ps < 1 || nj < 1 || n1 < 1) fail(PPC_SHAPE, "reshard_slices: extents must be positive");
        if (!recv || !out) fail(PPC_ARGUMENT, "reshard_slices: null pointer");
        // recv [r][slice][j][i] (block r: rank r's lateral columns of my
        // slices) -> out [slice][r*nj + j][i] (whole n1 x (G nj) slices)
        const size_t blk = sizeof(double) * (size_t)(nj * n1);
        for (int64_t r = 0; r < G; ++r)
            PPC_CUDA_CHECK(cudaMemcpy2DAsync(out + r * nj * n1, blk * (size_t)G, recv + r * ps * nj * n1, blk, blk,
                                             (size_t)ps, cudaMemcpyDeviceToDevice, stream()));
    });
}

int ppc_star_m_product(const double* A, int64_t n1, int64_t m, int64_t n3, const double* B, int64_t n2,
                       const double* M, double* C, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, m, n3);
        require_positive(n2, "n2");
        cudaStream_t s = stream();
        In a(A, n1 * m * n3, loc), b(B, m * n2 * n3, loc), mm(M, n3 * n3, loc);
        Out c(C, n1 * n2 * n3, loc);
        star_m(a.d, n1, m, n3, b.d, n2, mm.d, c.d, s);
        c.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_hosvd(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t k1, int64_t k2, int64_t k3,
              double* core, double* U1, double* U2, double* U3, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        if (k1 < 1 || k1 > n1 || k2 < 1 || k2 > n2 || k3 < 1 || k3 > n3)  // decompositions.cpp:230-233
            fail(PPC_ARGUMENT, "hosvd: multirank (" + std::to_string(k1) + "," + std::to_string(k2) + "," +
                                   std::to_string(k3) + ") outside the tensor extents");
        cudaStream_t s = stream();
        In a(A, n1 * n2 * n3, loc);
        Out c(core, k1 * k2 * k3, loc), u1(U1, n1 * k1, loc), u2(U2, n2 * k2, loc), u3(U3, n3 * k3, loc);
        hosvd(a.d, n1, n2, n3, k1, k2, k3, c.d, u1.d, u2.d, u3.d, s);
        c.finish();
        u1.finish();
        u2.finish();
        u3.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_hosvd_reconstruct(const double* core, int64_t k1, int64_t k2, int64_t k3, const double* U1, int64_t n1,
                          const double* U2, int64_t n2, const double* U3, int64_t n3, double* out, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        check_tensor(k1, k2, k3);
        if (k1 > n1 || k2 > n2 || k3 > n3) fail(PPC_SHAPE, "hosvd_reconstruct: core exceeds the factors");
        cudaStream_t s = stream();
        In c(core, k1 * k2 * k3, loc), u1(U1, n1 * k1, loc), u2(U2, n2 * k2, loc), u3(U3, n3 * k3, loc);
        Out o(out, n1 * n2 * n3, loc);
        hosvd_reconstruct(c.d, k1, k2, k3, u1.d, n1, u2.d, n2, u3.d, n3, o.d, s);
        o.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_matrix_svd_baseline(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t k, double* U,
                            double* S, double* V, double* error, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        const int64_t cap = std::min(n1 * n3, n2);
        if (k < 1 || k > cap)  // decompositions.cpp:248-251
            fail(PPC_ARGUMENT, "matrix_svd_baseline: k=" + std::to_string(k) + " outside [1," +
                                   std::to_string(cap) + "]");
        if (!error) fail(PPC_ARGUMENT, "null output");
        cudaStream_t s = stream();
        In a(A, n1 * n2 * n3, loc);
        Out u(U, n1 * n3 * k, loc), sv(S, k, loc), v(V, n2 * k, loc);
        *error = matrix_svd_baseline(a.d, n1, n2, n3, k, u.d, sv.d, v.d, s);
        u.finish();
        sv.finish();
        v.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_gram_plan(int64_t N, int64_t n3, int64_t* chunks, int64_t* chunk) {
    return guarded([&] {
        if (N < 1 || n3 < 1) fail(PPC_SHAPE, "gram_plan: extents must be positive");
        const GramPlan g = gram_plan(N, n3);
        *chunks = g.chunks;
        *chunk = g.chunk;
    });
}

int ppc_gram_partials(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk,
                      int64_t nchunks, double* parts, int loc) {
    return guarded([&] {
        validate_loc(loc);
        if (rows < 1 || n3 < 1 || ldT < rows || chunk < 1 || nchunks < 1)
            fail(PPC_SHAPE, "gram_partials: bad extents");
        if (chunk % 16) fail(PPC_ARGUMENT, "gram_partials: chunk must be a multiple of 16");
        cudaStream_t s = stream();
        In t(T, ldT * (n3 - 1) + rows, loc);
        Out o(parts, nchunks * n3 * n3, loc);
        gram_chunks(t.d, ldT, rows, n3, chunk, nchunks, o.d, s);
        o.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

namespace {
// Gram digits kept for the sharded forward transform, per thread.
thread_local std::map<int64_t, std::unique_ptr<OzakiDigits>> t_digits;
thread_local int64_t t_digits_next = 1;
}  // namespace

int ppc_gram_partials_keep(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk,
                           int64_t nchunks, double* parts, int64_t* handle, int* nonfinite) {
    return guarded([&] {
        if (!handle || !T || !parts || !nonfinite) fail(PPC_ARGUMENT, "null pointer");
        *handle = 0;
        *nonfinite = 0;
        if (rows < 1 || n3 < 1 || ldT < rows || chunk < 1 || nchunks < 1)
            fail(PPC_SHAPE, "gram_partials: bad extents");
        if (chunk % 16) fail(PPC_ARGUMENT, "gram_partials: chunk must be a multiple of 16");
        cudaStream_t s = stream();
        auto d = std::make_unique<OzakiDigits>();
        // the shard's finiteness (matrix_kernels.cpp:32), reported instead of
        // raised: the caller combines it over the ranks so all of them fail
        FiniteFlag nf(s);
        if (!gram_chunks(T, ldT, rows, n3, chunk, nchunks, parts, s, nf.d(), d.get())) {
            if (ldT == rows)  // the DMMA SYRK did not look: scan the block
                launch_nonfinite(T, rows * n3, nf.d(), s);
            else
                for (int64_t c = 0; c < n3; ++c) launch_nonfinite(T + c * ldT, rows, nf.d(), s);
        }
        PPC_CUDA_CHECK(cudaMemcpyAsync(nonfinite, nf.d(), sizeof(int), cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
        if (d->uniform && d->nd == 7) {
            *handle = t_digits_next++;
            t_digits[*handle] = std::move(d);
        }
    });
}

int ppc_mode3_forward_digits(int64_t handle, const double* Q, int64_t p, double* out) {
    return guarded([&] {
        auto it = t_digits.find(handle);
        if (it == t_digits.end()) fail(PPC_ARGUMENT, "mode3_forward_digits: unknown handle");
        if (!Q || !out) fail(PPC_ARGUMENT, "null pointer");
        const OzakiDigits& d = *it->second;
        const int64_t rows = d.rows;
        if (!ozaki_mode3_forward(d, rows, Q, p, out, stream()))
            fail(PPC_ARGUMENT, "mode3_forward_digits: shape not eligible");
    });
}

int ppc_digits_release(int64_t handle) {
    return guarded([&] { t_digits.erase(handle); });
}

int ppc_tree_reduce(double* parts, int64_t nparts, int64_t elems, int loc) {
    return guarded([&] {
        validate_loc(loc);
        if (nparts < 1 || elems < 1) fail(PPC_SHAPE, "tree_reduce: bad extents");
        cudaStream_t s = stream();
        In in(parts, nparts * elems, loc);
        double* d = const_cast<double*>(in.d);
        tree_reduce(d, nparts, elems, s);
        if (loc == PPC_HOST) {
            PPC_CUDA_CHECK(cudaMemcpyAsync(parts, d, sizeof(double) * elems, cudaMemcpyDeviceToHost, s));
            PPC_CUDA_CHECK(cudaStreamSynchronize(s));
        }
    });
}

int ppc_sym_eig_top(const double* G, int64_t n, int64_t p, double* Q, double* sigma, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_transform(n, p);
        cudaStream_t s = stream();
        In g(G, n * n, loc);
        Out q(Q, n * p, loc), sg(sigma, sigma ? p : 0, loc);
        eig_to_basis(g.d, n, p, q.d, sigma ? sg.d : nullptr, s);
        q.finish();
        if (sigma) sg.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

namespace {
thread_local std::map<int64_t, std::unique_ptr<EigSplit>> t_eig;
thread_local int64_t t_eig_next = 1;
EigSplit& eig_of(int64_t h) {
    auto it = t_eig.find(h);
    if (it == t_eig.end()) fail(PPC_ARGUMENT, "sym_eig_split: unknown handle");
    return *it->second;
}
}  // namespace

int ppc_sym_eig_split_begin(const double* G, int64_t n, int64_t p, int64_t* handle) {
    return guarded([&] {
        if (!G || !handle) fail(PPC_ARGUMENT, "null pointer");
        *handle = 0;
        check_transform(n, p);
        if (n <= kSubspaceMinN || !tridiag_eig_eligible(n, p)) return;  // caller: replicated ppc_sym_eig_top
        auto e = std::make_unique<EigSplit>(G, n, p, stream());
        *handle = t_eig_next++;
        t_eig[*handle] = std::move(e);
    });
}

int ppc_sym_eig_split_vectors(int64_t handle, int64_t j0, int64_t j1, double* Z) {
    return guarded([&] {
        if (!Z) fail(PPC_ARGUMENT, "null pointer");
        eig_of(handle).vectors(j0, j1, Z, stream());
    });
}

int ppc_sym_eig_split_finish(int64_t handle, double* Zall, int64_t j0, int64_t j1, double* Q) {
    return guarded([&] {
        if (!Zall || !Q) fail(PPC_ARGUMENT, "null pointer");
        EigSplit& e = eig_of(handle);
        e.finish(Zall, j0, j1, Q, stream());
        sign_rule(Q, e.n, j1 - j0, 1, nullptr, 0, stream());  // fix_svd_signs (matrix_kernels.cpp:35), per column
    });
}

int ppc_sym_eig_split_release(int64_t handle) {
    return guarded([&] { t_eig.erase(handle); });
}

int ppc_slice_residual_sums(const double* A, int64_t n1, int64_t n2, int64_t batch, int64_t k,
                            const double* U, const double* S, const double* V, double* sums, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, batch);
        check_spatial_rank(n1, n2, k, "slice_residual_sums");
        if (!sums) fail(PPC_ARGUMENT, "null output");
        cudaStream_t s = stream();
        In a(A, n1 * n2 * batch, loc), u(U, n1 * k * batch, loc), sv(S, k * batch, loc), v(V, n2 * k * batch, loc);
        DeviceBuffer out(sizeof(double) * 2);
        slice_residual_sums(a.d, n1, n2, batch, k, u.d, sv.d, v.d, out.d(), s);
        PPC_CUDA_CHECK(cudaMemcpyAsync(sums, out.d(), 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_gram_trace(const double* G, int64_t n, double* trace, int loc) {
    return guarded([&] {
        validate_loc(loc);
        require_positive(n, "n");
        if (!trace) fail(PPC_ARGUMENT, "null output");
        cudaStream_t s = stream();
        In g(G, n * n, loc);
        DeviceBuffer out(sizeof(double));
        gram_trace(g.d, n, out.d(), s);
        PPC_CUDA_CHECK(cudaMemcpyAsync(trace, out.d(), sizeof(double), cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int ppc_recon_residual_block(const double* A_blk, int64_t n1, int64_t nj, int64_t n3, int64_t ldA,
                             const double* U, const double* S, const double* V, int64_t n2,
                             int64_t j0, const double* Q, int64_t p, int64_t k, double* sums,
                             int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, nj, n3);
        check_transform(n3, p);
        if (j0 < 0 || j0 + nj > n2 || ldA < n1 * nj) fail(PPC_BOUNDS, "recon_residual_block: block outside the tensor");
        if (!sums) fail(PPC_ARGUMENT, "null output");
        cudaStream_t s = stream();
        In a(A_blk, ldA * (n3 - 1) + n1 * nj, loc), u(U, n1 * k * p, loc), sv(S, k * p, loc),
            v(V, n2 * k * p, loc), q(Q, n3 * p, loc);
        const auto r = recon_residual_block(a.d, n1, nj, n3, ldA, u.d, sv.d, v.d, n2, j0, q.d, p, k, s);
        sums[0] = r[0];
        sums[1] = r[1];
    });
}

int ppc_tsvdq_sweep(const double* A, int64_t n1, int64_t n2, int64_t n3, const int64_t* ps, int64_t np,
                    const int64_t* ks, int64_t nk, const double* Q, double* re, int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_tensor(n1, n2, n3);
        if (np < 1 || nk < 1 || !ps || !ks || !re) fail(PPC_ARGUMENT, "sweep: empty p or k grid");
        const int64_t kcap = std::min(n1, n2);
        int64_t pmax = 0, kmax = 0;
        for (int64_t i = 0; i < np; ++i) {  // tools/main.cpp:314-321 checks
            if (ps[i] < 1 || ps[i] > n3)
                fail(PPC_ARGUMENT, "p = " + std::to_string(ps[i]) + " exceeds n3 = " + std::to_string(n3));
            pmax = std::max(pmax, ps[i]);
        }
        for (int64_t i = 0; i < nk; ++i) {
            if (ks[i] < 1 || ks[i] > kcap)
                fail(PPC_ARGUMENT, "k = " + std::to_string(ks[i]) + " exceeds min(n1,n2) = " + std::to_string(kcap));
            kmax = std::max(kmax, ks[i]);
        }
        cudaStream_t s = stream();
        const int64_t N = n1 * n2;
        DeviceBuffer qbuf, abuf;
        const double* dQ;
        if (!Q && loc == PPC_HOST) {  // data-driven Q: the Gram overlaps the upload
            qbuf = DeviceBuffer(sizeof(double) * n3 * pmax);
            host_streamed_q(A, N, n3, pmax, abuf, qbuf.d(), nullptr, nullptr, nullptr, s);
            sweep_errors(abuf.d(), n1, n2, n3, qbuf.d(), pmax, kmax, ps, np, ks, nk, re, s);
            PPC_CUDA_CHECK(cudaStreamSynchronize(s));
            return;
        }
        In a(A, N * n3, loc);
        if (Q) {
            require_finite(a.d, N * n3, "svd", s);
            In qi(Q, n3 * pmax, loc);
            qbuf = DeviceBuffer(sizeof(double) * n3 * pmax);
            PPC_CUDA_CHECK(cudaMemcpyAsync(qbuf.d(), qi.d, sizeof(double) * n3 * pmax, cudaMemcpyDeviceToDevice, s));
        } else {
            qbuf = DeviceBuffer(sizeof(double) * n3 * pmax);
            data_q(a.d, N, n3, pmax, qbuf.d(), nullptr, s, true);
        }
        dQ = qbuf.d();
        sweep_errors(a.d, n1, n2, n3, dQ, pmax, kmax, ps, np, ks, nk, re, s);
    });
}

int ppc_tsvdq_compress(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t p, int64_t k,
                       double* Q, double* sigma, double* U, double* S, double* V, double* re,
                       int loc) {
    return guarded([&] {
        validate_loc(loc);
        check_transform(n3, p);
        check_tensor(n1, n2, n3);
        check_spatial_rank(n1, n2, k, "tsvdq");
        if (!re) fail(PPC_ARGUMENT, "null output");
        cudaStream_t s = stream();
        const int64_t N = n1 * n2;
        Out q(Q, n3 * p, loc), sg(sigma, sigma ? p : 0, loc), u(U, n1 * k * p, loc),
            sv(S, k * p, loc), v(V, n2 * k * p, loc);
        DeviceBuffer abuf, est(sizeof(double) * 4);  // trace(G), slice residual, ||Ahat||^2
        OzakiDigits tdig;  // A's 7-digit Gram split, reused by the forward transform
        const double* dA = A;
        if (loc == PPC_HOST) {
            host_streamed_q(A, N, n3, p, abuf, q.d, sigma ? sg.d : nullptr, est.d(), &tdig, s);
            dA = abuf.d();
        } else {
            data_q(dA, N, n3, p, q.d, sigma ? sg.d : nullptr, s, true, est.d(), &tdig);
        }
        tsvdq(dA, n1, n2, n3, q.d, p, k, u.d, sv.d, v.d, s, est.d() + 1, &tdig, est.d());
        tdig = OzakiDigits();  // the 7-digit split of A (30 GB at cfg5) is not needed past the transform
        *re = compress_relative_error(dA, n1, n2, n3, u.d, sv.d, v.d, q.d, p, k, est.d(), s);
        q.finish();
        if (sigma) sg.finish();
        u.finish();
        sv.finish();
        v.finish();
        if (loc == PPC_HOST) PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
