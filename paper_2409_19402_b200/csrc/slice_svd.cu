// Facewise SVD, Gram SYRK and the data-driven basis Q.
//
//   slice_svd  — matrix_kernels.cpp:29-37 per transform-domain slice
//                (decompositions.cpp:75-81). Small slices: one-CTA Jacobi (K6).
//   gram       — G = T^T T with deterministic split-K over pixel chunks and a
//                fixed pairwise tree over chunks (K4).
//   data_q     — transforms.cpp:97-115 via Gram + symmetric eigensolve (K5).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "dmma_gemm.cuh"
#include "engine.h"
#include "internal.h"
#include "jacobi.cuh"
#include "kernels.cuh"
#include "ozaki.h"
#include "slice_svd.cuh"

namespace ppc {

namespace {

__global__ void tree_add_kernel(double* parts, int64_t nparts, int64_t elems, int64_t width) {
    // parts[s] += parts[s + width] for s multiple of 2*width
    const int64_t total = ((nparts + 2 * width - 1) / (2 * width)) * elems;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t grp = i / elems, e = i % elems;
        const int64_t a = grp * 2 * width, b = a + width;
        if (b < nparts) parts[a * elems + e] += parts[b * elems + e];
    }
}

// Tb = T re-laid as consecutive blocks of KB rows: block kb is the KB x n3
// column-major matrix of rows [kb*KB, kb*KB + KB) (zero-padded at the end).
__global__ void block_rows_kernel(const double* __restrict__ T, double* __restrict__ Tb, int64_t N,
                                  int64_t ldT, int64_t n3, int kshift, int64_t total) {
    const int64_t KB = 1LL << kshift;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int64_t kb = e / (KB * n3), rem = e - kb * KB * n3;
        const int64_t a = rem >> kshift, ii = rem & (KB - 1);
        const int64_t i = (kb << kshift) + ii;
        Tb[e] = i < N ? T[i + a * ldT] : 0.0;
    }
}

__global__ void sqrt_clamp_kernel(const double* lam, double* sig, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) sig[i] = sqrt(fmax(lam[i], 0.0));
}

}  // namespace

GramPlan gram_plan(int64_t N, int64_t n3) {
    // Chunk count depends on (N, n3) only — never on the device count — so
    // the reduction tree (and hence Q) is bitwise identical on 1..8 GPUs.
    GramPlan g;
    const int64_t bt = n3 <= 32 ? 1 : (n3 + 127) / 128;
    const int64_t tiles = std::max<int64_t>(1, bt * (bt + 1) / 2);
    int64_t want = std::max<int64_t>(1, (4 * 148) / tiles);
    int64_t maxc = std::max<int64_t>(1, N / 512);
    int64_t c = 1;
    while (c * 2 <= want && c * 2 <= maxc) c *= 2;
    // the INT8 Ozaki SYRK wants chunks of >= 4096 rows (one digit block
    // each); it is far faster than a wide split-K DMMA SYRK on short Grams
    if (ozaki_path_on() && n3 >= 128 && N >= 4 * 4096)
        while (c > 1 && (N + c - 1) / c < 4096) c /= 2;
    g.chunks = c;
    g.chunk = ((N + c - 1) / c + 15) / 16 * 16;
    return g;
}

void gram_partials(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk,
                   int64_t chunks, double* parts, cudaStream_t s, int kshift) {
    GemmDesc d;
    d.M = n3; d.N = n3; d.K = rows;
    d.A = T; d.lda = ldT; d.a_kmajor = true;   // A(m,k) = T[k + m*ldT]
    d.B = T; d.ldb = ldT; d.b_nmajor = false;  // B(k,n) = T[k + n*ldT]
    d.C = parts; d.ldc = n3;
    d.symmetric = true;
    d.splits = chunks;
    d.kchunk = chunk;
    d.strideCsplit = n3 * n3;
    if (kshift) {  // T is in the row-blocked layout (block_rows_kernel)
        d.kshift = kshift;
        d.kbstride = (1LL << kshift) * n3;
        d.lda = d.ldb = 1LL << kshift;
    }
    gemm(d, s);
}

void tree_reduce(double* parts, int64_t nparts, int64_t elems, cudaStream_t s) {
    for (int64_t w = 1; w < nparts; w *= 2) {
        const int64_t total = ((nparts + 2 * w - 1) / (2 * w)) * elems;
        const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
        tree_add_kernel<<<grid, 256, 0, s>>>(parts, nparts, elems, w);
        count_launch();
        check_launch("tree_add");
    }
}

// Partial Grams of `nchunks` consecutive chunks of `chunk` rows of T (rows x
// n3, leading dimension ldT) into parts (nchunks x n3 x n3).
bool gram_chunks(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk,
                 int64_t nchunks, double* parts, cudaStream_t s, int* nonfinite, OzakiDigits* keep,
                 int64_t block_base, int64_t total_blocks) {
    // INT8 tensor-core (Ozaki) path for large Grams; it reads T column by
    // column, so no re-layout either
    if (ozaki_gram_partials(T, ldT, rows, n3, chunk, nchunks, parts, s, nonfinite, keep, block_base, total_blocks))
        return nonfinite != nullptr;
    // Large tube matrices: each SYRK pipeline stage would touch one 2 MB page
    // per column (columns are ldT*8 bytes apart), thrashing the TLB. Re-lay T
    // into 2048-row blocks first (one extra HBM pass); same summation order.
    static const bool no_relayout = std::getenv("PPC_NO_RELAYOUT") != nullptr;
    const int kshift = (!no_relayout && ldT >= (1LL << 20) && n3 >= 64) ? 11 : 0;
    DeviceBuffer tb;
    const double* src = T;
    int64_t ld = ldT;
    if (kshift) {
        StageTimer tr("gram_relayout", s, 0.0, 16.0 * rows * n3);
        const int64_t KB = 1LL << kshift, nb = (rows + KB - 1) / KB;
        tb = DeviceBuffer(sizeof(double) * nb * KB * n3);
        const int64_t total = nb * KB * n3;
        block_rows_kernel<<<148 * 16, 256, 0, s>>>(T, tb.d(), rows, ldT, n3, kshift, total);
        count_launch();
        check_launch("block_rows");
        src = tb.d();
        ld = KB;
    }
    gram_partials(src, ld, rows, n3, chunk, nchunks, parts, s, kshift);
    return false;
}

bool gram(const double* T, int64_t N, int64_t n3, double* G, cudaStream_t s, int* nonfinite, OzakiDigits* keep) {
    StageTimer tm("gram_syrk", s, (double)N * n3 * n3, 8.0 * N * n3);
    const GramPlan g = gram_plan(N, n3);
    if (g.chunks == 1) return gram_chunks(T, N, N, n3, g.chunk, 1, G, s, nonfinite, keep);
    DeviceBuffer parts(sizeof(double) * g.chunks * n3 * n3);
    const bool checked = gram_chunks(T, N, N, n3, g.chunk, g.chunks, parts.d(), s, nonfinite, keep);
    tree_reduce(parts.d(), g.chunks, n3 * n3, s);
    PPC_CUDA_CHECK(cudaMemcpyAsync(G, parts.d(), sizeof(double) * n3 * n3, cudaMemcpyDeviceToDevice, s));
    return checked;
}

FiniteFlag::FiniteFlag(cudaStream_t s) : flag(status_words()) {
    PPC_CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int), s));
}

void FiniteFlag::check(cudaStream_t s, const char* who) {
    int h = 0;
    PPC_CUDA_CHECK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    if (h) fail(PPC_NUMERIC, std::string(who) + ": input has non-finite entries");
}

void sym_eig_top(const double* G, int64_t n, int64_t p, double* Q, double* lambda, cudaStream_t s,
                 bool accurate_vectors) {
    // One-sided Jacobi on the PSD G: V = eigenvectors, column norms of G V =
    // eigenvalues, descending (stable order on ties).
    if (n <= kSubspaceMinN) {
        jacobi_svd(G, n, n, n * n, 1, p, nullptr, lambda, Q, nullptr, s);
        return;
    }
    // one matrix: direct Householder tridiagonalization + bisection +
    // inverse iteration (tridiag_eig.cu) instead of the subspace iteration
    if (tridiag_eig_eligible(n, p)) {
        tridiag_eig_top(G, n, p, Q, lambda, s);
        return;
    }
    subspace_eig_top(G, n, 1, p, Q, lambda, s, accurate_vectors);
}

void eig_to_basis(const double* G, int64_t n3, int64_t p, double* Q, double* sigma, cudaStream_t s,
                  bool accurate_vectors) {
    DeviceBuffer lam(sizeof(double) * n3);
    {
        StageTimer tm("eig_q", s);
        sym_eig_top(G, n3, p, Q, lam.d(), s, accurate_vectors);
    }
    sign_rule(Q, n3, p, 1, nullptr, 0, s);  // fix_svd_signs on U3 (matrix_kernels.cpp:35)
    if (sigma) {
        sqrt_clamp_kernel<<<(unsigned)((p + 255) / 256), 256, 0, s>>>(lam.d(), sigma, p);
        count_launch();
        check_launch("sqrt_clamp");
    }
}

namespace {
__global__ void trace_kernel(const double* __restrict__ G, int64_t n, double* __restrict__ out) {
    __shared__ double red[32];
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += G[i + i * n];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
        a = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (threadIdx.x == 0) *out = a;
    }
}
}  // namespace

void gram_trace(const double* G, int64_t n, double* out, cudaStream_t s) {
    trace_kernel<<<1, 256, 0, s>>>(G, n, out);
    count_launch();
    check_launch("trace");
}

bool data_q(const double* T, int64_t N, int64_t n3, int64_t p, double* Q, double* sigma,
            cudaStream_t s, bool check_finite, double* gtrace, OzakiDigits* keep) {
    DeviceBuffer G(sizeof(double) * n3 * n3);
    if (check_finite) {
        FiniteFlag nf(s);
        if (gram(T, N, n3, G.d(), s, nf.d(), keep))
            nf.check(s, "svd");
        else
            require_finite(T, N * n3, "svd", s);
    } else {
        gram(T, N, n3, G.d(), s, nullptr, keep);
    }
    if (gtrace) gram_trace(G.d(), n3, gtrace, s);
    // When p > min(n3, N) the unfolding has only min(n3, N) singular vectors;
    // the eigenvectors of G for its zero eigenvalues complete the basis
    // (transforms.cpp:104-111 pads with an orthonormal completion).
    eig_to_basis(G.d(), n3, p, Q, sigma, s);
    return p > std::min(n3, N);
}

void slice_svd(const double* A, int64_t m, int64_t n, int64_t stride, int64_t batch, int64_t k,
               double* U, double* S, double* V, double* tail2, cudaStream_t s, const char* finite_who) {
    const int64_t r = std::min(m, n);
    const bool sub = !(r <= kSubspaceMinN || jacobi_smem_bytes(m, n) <= 200 * 1024) && !(k > r / 2);
    if (finite_who && !(sub && m >= n && ozaki_path_on())) {  // no INT8 slice-Gram split to ride on
        if (stride != m * n) fail(PPC_ARGUMENT, "slice_svd: the finiteness check needs contiguous slices");
        require_finite(A, m * n * batch, finite_who, s);  // matrix_kernels.cpp:32
        finite_who = nullptr;
    }
    if (r <= kSubspaceMinN || jacobi_smem_bytes(m, n) <= 200 * 1024) {
        jacobi_svd(A, m, n, stride, batch, k, U, S, V, tail2, s);
        return;
    }
    if (k > r / 2) {  // most of the spectrum (tsvdq2: all of it): blocked one-sided Jacobi
        if (block_jacobi_eligible(m, n, k))
            block_jacobi_svd(A, m, n, stride, batch, k, U, S, V, tail2, s);
        else
            jacobi_svd(A, m, n, stride, batch, k, U, S, V, tail2, s);
        return;
    }
    if (!subspace_svd(A, m, n, stride, batch, k, U, S, V, tail2, s, finite_who) && finite_who) {
        // the INT8 split did not run after all (shape not eligible): its checks
        // were skipped, so check now (results are discarded on failure)
        require_finite(A, m * n * batch, finite_who, s);
    }
}

}  // namespace ppc
