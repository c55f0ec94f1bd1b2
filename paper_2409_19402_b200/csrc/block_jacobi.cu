// K6b — batched block one-sided Jacobi SVD for large slices with a large k.
//
// The full (or nearly full) SVD of slices too large for the one-CTA Jacobi
// kernel (K6): tsvdq2 keeps k = min(n1, n2) triplets of every slice
// (decompositions.cpp:120-209 needs the whole spectrum), and the Gram +
// subspace route (K7) is only for k <= r/2. Eigen's JacobiSVD
// (matrix_kernels.cpp:29-37) is one-sided Jacobi; this is its blocked form:
//
//   W = A (R x C, R >= C; a wide slice is transposed first), columns padded to
//   2B blocks of 32, V = I. A sweep runs 2B-1 rounds of the round-robin block
//   pairing; in a round every pair (a, c) of every slice:
//     1. G = [W_a W_c]^T [W_a W_c]  (64 x 64, fixed-order FP64 sums)  — bj_gram
//     2. G = J diag J^T by the one-CTA Jacobi eigensolver (K6, eigen mode)
//     3. [W_a W_c] <- [W_a W_c] J,  [V_a V_c] <- [V_a V_c] J           — bj_apply
//   skipping pairs whose columns are already orthogonal to working precision
//   (|G_ij| <= tol sqrt(G_ii G_jj), tol = eps sqrt(R)). Sweeps repeat until no
//   pair of a slice rotates (one host read per sweep).
//   Then sigma_j = ||W_j||, U_j = W_j / sigma_j, descending with a stable
//   (index) tie-break, the sign rule (matrix_kernels.cpp:16-25), and an
//   orthonormal completion of U and V for zero singular values (as K6).
//
// Every dot product is recomputed from the rotated columns each round, so the
// stopping test is the one-sided Jacobi test on the actual columns; all sums
// have a fixed order, so results are deterministic and independent of how
// many slices share the launch.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.h"
#include "jacobi.cuh"
#include "kernels.cuh"
#include "slice_svd.cuh"

namespace ppc {

namespace {

constexpr int kBW = 32;          // block width (columns)
constexpr int kPW = 2 * kBW;     // pair width
constexpr int kGramRows = 64;    // row tile of the Gram kernel
constexpr int kApplyRows = 256;  // rows per CTA of the apply kernel

__device__ __forceinline__ void rr_pair(int r, int pi, int P, int& a, int& c) {
    if (pi == 0) {
        a = r;
        c = P - 1;
    } else {
        const int m = P - 1;
        a = r + pi;
        if (a >= m) a -= m;
        c = r + m - pi;
        if (c >= m) c -= m;
    }
    if (a > c) {
        const int t = a;
        a = c;
        c = t;
    }
}

// column l (0..63) of the pair (a, c) -> column index of W / V
__device__ __forceinline__ int pair_col(int l, int a, int c) { return l < kBW ? a * kBW + l : c * kBW + (l - kBW); }

// W (R x Cp per slice) = A (tall) or A^T (wide), zero padding columns; V = I (Cp x Cp).
__global__ void bj_init_kernel(const double* __restrict__ A, int64_t m, int64_t n, int64_t strideA, int64_t R,
                               int64_t C, int64_t Cp, double* __restrict__ W, double* __restrict__ V) {
    const int64_t b = blockIdx.y;
    const double* a = A + b * strideA;
    double* w = W + b * R * Cp;
    double* v = V + b * Cp * Cp;
    const bool tall = m >= n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < R * Cp; e += stride) {
        const int64_t i = e % R, j = e / R;
        w[e] = j < C ? (tall ? a[i + j * m] : a[j + i * m]) : 0.0;
    }
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < Cp * Cp; e += stride)
        v[e] = (e % Cp) == (e / Cp) ? 1.0 : 0.0;
}

// G (64 x 64, column-major) of pair pi of round r for slice blockIdx.y, and
// the pair's largest scaled off-diagonal |G_ij| / sqrt(G_ii G_jj).
__global__ void __launch_bounds__(256) bj_gram_kernel(const double* __restrict__ W, int64_t R, int64_t Cp, int P,
                                                      int r, double* __restrict__ G, double* __restrict__ off) {
    __shared__ double tile[kGramRows * (kPW + 1)];  // [row][col], padded row stride
    __shared__ double red[8];
    const int pi = blockIdx.x;
    const int64_t b = blockIdx.y;
    int a, c;
    rr_pair(r, pi, P, a, c);
    const double* w = W + b * R * Cp;
    const int tid = threadIdx.x;
    const int i = tid & (kPW - 1), jg = tid >> 6;  // this thread: G(i, jg*16 .. jg*16+15)
    double acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = 0.0;
    for (int64_t r0 = 0; r0 < R; r0 += kGramRows) {
        __syncthreads();
        for (int e = tid; e < kGramRows * kPW; e += 256) {
            const int rr = e % kGramRows, l = e / kGramRows;
            const int64_t row = r0 + rr;
            tile[rr * (kPW + 1) + l] = row < R ? w[row + (int64_t)pair_col(l, a, c) * R] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int rr = 0; rr < kGramRows; ++rr) {
            const double x = tile[rr * (kPW + 1) + i];
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] = fma(x, tile[rr * (kPW + 1) + jg * 16 + q], acc[q]);
        }
    }
    double* g = G + ((int64_t)b * gridDim.x + pi) * kPW * kPW;
#pragma unroll
    for (int q = 0; q < 16; ++q) g[i + (jg * 16 + q) * kPW] = acc[q];
    // scaled off-diagonal: the diagonal comes from the threads that own it
    __syncthreads();
    __shared__ double dg[kPW];
#pragma unroll
    for (int q = 0; q < 16; ++q)
        if (i == jg * 16 + q) dg[i] = acc[q];
    __syncthreads();
    double mx = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int j = jg * 16 + q;
        if (j != i) {
            const double d = dg[i] * dg[j];
            if (d > 0.0) mx = fmax(mx, fabs(acc[q]) / sqrt(d));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
        for (int q = 1; q < 8; ++q) mx = fmax(mx, red[q]);
        off[(int64_t)b * gridDim.x + pi] = fmax(mx, red[0]);
    }
}

// [X_a X_c] <- [X_a X_c] J for the rows of X = W (R rows) then V (Cp rows)
// handled by this CTA (blockIdx.z), if the pair rotates at all.
__global__ void __launch_bounds__(256) bj_apply_kernel(double* __restrict__ W, double* __restrict__ V, int64_t R,
                                                       int64_t Cp, int P, int r, const double* __restrict__ J,
                                                       const double* __restrict__ off, double tol,
                                                       unsigned long long* __restrict__ rotated) {
    extern __shared__ double sm[];
    double* j_s = sm;                 // J, [l][jj] column-major 64 x 64
    double* x_s = sm + kPW * kPW;     // rows x 64, [l][row]
    const int pi = blockIdx.x;
    const int64_t b = blockIdx.y;
    const int64_t pid = b * gridDim.x + pi;
    if (!(off[pid] > tol)) return;
    int a, c;
    rr_pair(r, pi, P, a, c);
    const int tid = threadIdx.x;
    if (blockIdx.z == 0 && tid == 0) rotated[b] = 1ull;
    const double* jm = J + pid * kPW * kPW;
    for (int e = tid; e < kPW * kPW; e += 256) j_s[e] = jm[e];
    // the CTA's rows: chunk z of W's rows, then of V's rows
    const int64_t zw = (R + kApplyRows - 1) / kApplyRows;
    double* base;
    int64_t ld, lr0, nrows;
    if ((int64_t)blockIdx.z < zw) {
        base = W + b * R * Cp;
        ld = R;
        lr0 = (int64_t)blockIdx.z * kApplyRows;
        nrows = std::min<int64_t>(kApplyRows, R - lr0);
    } else {
        base = V + b * Cp * Cp;
        ld = Cp;
        lr0 = ((int64_t)blockIdx.z - zw) * kApplyRows;
        nrows = std::min<int64_t>(kApplyRows, Cp - lr0);
    }
    for (int e = tid; e < kApplyRows * kPW; e += 256) {
        const int rr = e % kApplyRows, l = e / kApplyRows;
        x_s[l * kApplyRows + rr] = rr < nrows ? base[lr0 + rr + (int64_t)pair_col(l, a, c) * ld] : 0.0;
    }
    __syncthreads();
    if (tid < nrows) {
        double acc[kPW];
#pragma unroll
        for (int q = 0; q < kPW; ++q) acc[q] = 0.0;
#pragma unroll 4
        for (int l = 0; l < kPW; ++l) {
            const double x = x_s[l * kApplyRows + tid];
#pragma unroll
            for (int q = 0; q < kPW; ++q) acc[q] = fma(x, j_s[l + q * kPW], acc[q]);
        }
#pragma unroll
        for (int q = 0; q < kPW; ++q) base[lr0 + tid + (int64_t)pair_col(q, a, c) * ld] = acc[q];
    }
}

// per slice: sigma_j = ||W_j||, stable descending order, the leading k
// triplets; zero singular values get U, V by orthonormal completion.
__global__ void __launch_bounds__(256) bj_finalize_kernel(const double* __restrict__ W, const double* __restrict__ V,
                                                          int64_t R, int64_t C, int64_t Cp, int64_t k, bool tall,
                                                          double* __restrict__ U, double* __restrict__ S,
                                                          double* __restrict__ Vo, double* __restrict__ tail2,
                                                          double* __restrict__ nrm, int* __restrict__ order,
                                                          int64_t m, int64_t n) {
    const int64_t b = blockIdx.x;
    const double* w = W + b * R * Cp;
    const double* v = V + b * Cp * Cp;
    double* nb = nrm + b * Cp;
    int* ob = order + b * Cp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int64_t j = warp; j < Cp; j += nw) {
        double s = 0.0;
        for (int64_t i = lane; i < R; i += 32) s = fma(w[i + j * R], w[i + j * R], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        // padding columns (V support outside the C real rows) never hold
        // content; rank them behind every real column
        if (lane == 0) nb[j] = sqrt(s);
    }
    __syncthreads();
    // rank of column j: count of columns before it in (descending sigma, ascending index)
    for (int64_t j = tid; j < Cp; j += blockDim.x) {
        const double sj = nb[j];
        int64_t rk = 0;
        for (int64_t q = 0; q < Cp; ++q) {
            const double sq = nb[q];
            rk += (sq > sj) || (sq == sj && q < j);
        }
        ob[rk] = (int)j;
    }
    __syncthreads();
    // outputs: slice-major, U (m x k), S (k), V (n x k) in the caller's roles
    double* Ub = U + b * m * k;
    double* Vb = Vo + b * n * k;
    double* Sb = S + b * k;
    for (int64_t q = warp; q < k; q += nw) {
        const int j = ob[q];
        const double sg = nb[j];
        const double inv = sg > 0.0 ? 1.0 / sg : 0.0;
        if (lane == 0) Sb[q] = sg;
        // left vectors of W: W_j / sigma (length R); right: V_j (length C)
        double* left = tall ? Ub + q * m : Vb + q * n;
        double* right = tall ? Vb + q * n : Ub + q * m;
        for (int64_t i = lane; i < R; i += 32) left[i] = w[i + (int64_t)j * R] * inv;
        for (int64_t i = lane; i < C; i += 32) right[i] = sg > 0.0 ? v[i + (int64_t)j * Cp] : 0.0;
    }
    if (tail2 && tid == 0) {
        double t = 0.0;
        for (int64_t q = k; q < C; ++q) t += nb[ob[q]] * nb[ob[q]];
        tail2[b] = t;
    }
}

// Orthonormal completion of the zero-sigma columns of X (rows x k per slice):
// e_t with t the row of least captured mass, projected out of the other
// columns twice (CGS2) and normalized; columns in ascending order.
__global__ void __launch_bounds__(256) complete_zero_kernel(double* __restrict__ X, int64_t rows, int64_t k,
                                                            const double* __restrict__ S,
                                                            double* __restrict__ rowm) {
    const int64_t b = blockIdx.x;
    const double* sb = S + b * k;
    bool any = false;
    for (int64_t q = 0; q < k; ++q) any |= !(sb[q] > 0.0);
    if (!any) return;
    double* x = X + b * rows * k;
    double* rm = rowm + b * rows;
    __shared__ double red[33];
    extern __shared__ double cf[];  // k projection coefficients
    __shared__ int64_t tmin;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    auto bsum = [&](double v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __syncthreads();
        if (lane == 0) red[warp] = v;
        __syncthreads();
        if (warp == 0) {
            double a = lane < nw ? red[lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (lane == 0) red[32] = a;
        }
        __syncthreads();
        return red[32];
    };
    for (int64_t t = tid; t < rows; t += blockDim.x) {
        double s = 0.0;
        for (int64_t q = 0; q < k; ++q)
            if (sb[q] > 0.0) s = fma(x[t + q * rows], x[t + q * rows], s);
        rm[t] = s;
    }
    __syncthreads();
    for (int64_t j = 0; j < k; ++j) {
        if (sb[j] > 0.0) continue;
        if (tid == 0) {
            int64_t best = 0;
            for (int64_t t = 1; t < rows; ++t)
                if (rm[t] < rm[best]) best = t;
            tmin = best;
        }
        __syncthreads();
        double* v = x + j * rows;
        for (int64_t t = tid; t < rows; t += blockDim.x) v[t] = t == tmin ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass) {
            __syncthreads();
            for (int64_t q = warp; q < k; q += nw) {
                double a = 0.0;
                if (q != j && (sb[q] > 0.0 || q < j))
                    for (int64_t t = lane; t < rows; t += 32) a = fma(x[t + q * rows], v[t], a);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (lane == 0) cf[q] = (q != j && (sb[q] > 0.0 || q < j)) ? a : 0.0;
            }
            __syncthreads();
            for (int64_t t = tid; t < rows; t += blockDim.x) {
                double y = v[t];
                for (int64_t q = 0; q < k; ++q) y = fma(-x[t + q * rows], cf[q], y);
                v[t] = y;
            }
        }
        double a = 0.0;
        for (int64_t t = tid; t < rows; t += blockDim.x) a = fma(v[t], v[t], a);
        const double nv = bsum(a);
        const double inv = nv > 0.0 ? 1.0 / sqrt(nv) : 0.0;
        for (int64_t t = tid; t < rows; t += blockDim.x) {
            v[t] *= inv;
            rm[t] = fma(v[t], v[t], rm[t]);
        }
        __syncthreads();
    }
}

}  // namespace

bool block_jacobi_eligible(int64_t m, int64_t n, int64_t k) {
    const int64_t C = std::min(m, n);
    return k <= C && C >= 2 * kBW && C <= 8192;
}

void block_jacobi_svd(const double* A, int64_t m, int64_t n, int64_t strideA, int64_t batch, int64_t k, double* U,
                      double* S, double* V, double* tail2, cudaStream_t s) {
    const bool tall = m >= n;
    const int64_t R = tall ? m : n, C = tall ? n : m;
    const int64_t Cp = (C + kPW - 1) / kPW * kPW;
    const int P = (int)(Cp / kBW), B = P / 2;  // blocks, pairs per round
    StageTimer tm("block_jacobi", s, 0.0, 8.0 * batch * m * n);
    DeviceBuffer W(sizeof(double) * batch * R * Cp), Vw(sizeof(double) * batch * Cp * Cp),
        G(sizeof(double) * batch * B * kPW * kPW), J(sizeof(double) * batch * B * kPW * kPW),
        lam(sizeof(double) * batch * B * kPW), off(sizeof(double) * batch * B), rot(sizeof(unsigned long long) * batch);
    bj_init_kernel<<<dim3(148, (unsigned)batch), 256, 0, s>>>(A, m, n, strideA, R, C, Cp, W.d(), Vw.d());
    count_launch();
    check_launch("bj_init");
    const double tol = 2.220446049250313e-16 * std::sqrt((double)R);
    const size_t asm_bytes = sizeof(double) * (kPW * kPW + kApplyRows * kPW);
    PPC_CUDA_CHECK(cudaFuncSetAttribute(bj_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)asm_bytes));
    const unsigned zchunks = (unsigned)((R + kApplyRows - 1) / kApplyRows + (Cp + kApplyRows - 1) / kApplyRows);
    std::vector<unsigned long long> h((size_t)batch);
    static const bool dbg = std::getenv("PPC_JACOBI_DEBUG") != nullptr;
    int sweep = 0;
    for (; sweep < 40; ++sweep) {
        PPC_CUDA_CHECK(cudaMemsetAsync(rot.d(), 0, sizeof(unsigned long long) * batch, s));
        for (int r = 0; r < P - 1; ++r) {
            bj_gram_kernel<<<dim3((unsigned)B, (unsigned)batch), 256, 0, s>>>(W.d(), R, Cp, P, r, G.d(), off.d());
            count_launch();
            check_launch("bj_gram");
            jacobi_svd(G.d(), kPW, kPW, kPW * kPW, batch * B, kPW, nullptr, lam.d(), J.d(), nullptr, s);
            bj_apply_kernel<<<dim3((unsigned)B, (unsigned)batch, zchunks), 256, asm_bytes, s>>>(
                W.d(), Vw.d(), R, Cp, P, r, J.d(), off.d(), tol, rot.as<unsigned long long>());
            count_launch();
            check_launch("bj_apply");
        }
        PPC_CUDA_CHECK(cudaMemcpyAsync(h.data(), rot.d(), sizeof(unsigned long long) * batch,
                                       cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
        bool any = false;
        for (auto v : h) any |= v != 0;
        if (!any) break;
    }
    if (dbg)
        fprintf(stderr, "[block-jacobi] %lldx%lld batch %lld k %lld sweeps %d\n", (long long)m, (long long)n,
                (long long)batch, (long long)k, sweep + 1);
    DeviceBuffer nrm(sizeof(double) * batch * Cp), ord(sizeof(int) * batch * Cp),
        rowm(sizeof(double) * batch * std::max(m, n));
    bj_finalize_kernel<<<(unsigned)batch, 256, 0, s>>>(W.d(), Vw.d(), R, C, Cp, k, tall, U, S, V, tail2, nrm.d(),
                                                      ord.as<int>(), m, n);
    count_launch();
    check_launch("bj_finalize");
    const size_t czs = sizeof(double) * (size_t)k;  // k <= 8192: <= 64 KB
    if (czs > 48 * 1024)
        PPC_CUDA_CHECK(cudaFuncSetAttribute(complete_zero_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)czs));
    complete_zero_kernel<<<(unsigned)batch, 256, czs, s>>>(U, m, k, S, rowm.d());
    count_launch();
    complete_zero_kernel<<<(unsigned)batch, 256, czs, s>>>(V, n, k, S, rowm.d());
    count_launch();
    check_launch("complete_zero");
    sign_rule(U, m, k, batch, V, n, s);  // matrix_kernels.cpp:16-25
}

}  // namespace ppc
