// K5/K7 — top-k symmetric eigensolver and large-slice SVD.
//
// For slices too large for the one-CTA Jacobi kernel (K6) the facewise SVD
// (matrix_kernels.cpp:29-37 applied per slice, decompositions.cpp:75-81)
// runs as:
//   1. batched Gram SYRK  G_i = A_i^T A_i  (or A_i A_i^T when wide)   [DMMA]
//   2. top-k eigenvectors of every G_i by Chebyshev-filtered subspace
//      iteration with Rayleigh-Ritz, prefix locking and operator deflation
//      (G - X_L Theta_L X_L^T), a per-slice polynomial degree that bounds the
//      amplification spread inside the active block, and CholQR2 (with a
//      shift on the first pass) for orthonormalization            [DMMA]
//   3. Rayleigh-Ritz polish on A itself: W = A V_k, one-sided Jacobi SVD of
//      W -> U, sigma and the k x k rotation of V_k. This restores singular
//      values to ~eps * sigma_1 absolute accuracy (the Gram route alone loses
//      relative accuracy as (sigma_1/sigma_j)^2).
// Every GEMM-shaped step is a batched call of the FP64 DMMA GEMM; the small
// per-slice dense work (Cholesky + triangular inverse, b x b eigensolve) runs
// one CTA per slice. The host drives the iteration and reads back only the
// b Ritz values and residual norms per slice per iteration.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "dmma_gemm.cuh"
#include "engine.h"
#include "internal.h"
#include "jacobi.cuh"
#include "kernels.cuh"
#include "ozaki.h"
#include "panel.cuh"
#include "slice_svd.cuh"

namespace ppc {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Deterministic N(0,1) start block (counter-based, Box-Muller).
__global__ void randn_kernel(double* X, int64_t n, uint64_t seed) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t a = mix64(seed ^ (2 * (uint64_t)i)), b = mix64(seed ^ (2 * (uint64_t)i + 1));
        const double u1 = ((a >> 11) + 1) * 0x1.0p-53, u2 = (b >> 11) * 0x1.0p-53;
        X[i] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    }
}

// Y_next = a*Z + b*Y + c*Yp with per-slice coefficients coef[3*slice + {0,1,2}];
// columns below c0 (locked in every filtered slice) just carry Y.
// zmap (nullable): element block z of the launch is slice zmap[z] (only the
// slices still filtering at this degree; the others keep their own Y).
__global__ void cheb_kernel(double* __restrict__ Yn, const double* __restrict__ Z,
                            const double* __restrict__ Y, const double* __restrict__ Yp,
                            const double* __restrict__ coef, int64_t per_slice, int64_t total,
                            int64_t r, int64_t c0, const int* __restrict__ zmap) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t ii = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ii < total; ii += stride) {
        const int64_t z = ii / per_slice, off = ii - z * per_slice;
        const int64_t s = zmap ? (int64_t)zmap[z] : z;
        const int64_t i = s * per_slice + off;
        if (off / r < c0) {
            Yn[i] = Y[i];
            continue;
        }
        const double a = coef[3 * s], b = coef[3 * s + 1], c = coef[3 * s + 2];
        double v = b * Y[i];
        if (a != 0.0) v += a * Z[i];  // frozen slices: Z is not computed for them
        if (c != 0.0) v += c * Yp[i];
        Yn[i] = v;
    }
}

// P(i, j, s) *= w(i, s)   (rows of the lp x cols block scaled: Theta_L mask;
// w has stride b per slice)
// coef (nullable): also times the slice's Chebyshev coefficient a = coef[3 s]
__global__ void scale_rows_kernel(double* P, const double* w, int64_t lp, int64_t b, int64_t cols, int64_t total,
                                  const double* __restrict__ coef) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t row = i % lp, s = i / (lp * cols);
        P[i] *= coef ? w[row + s * b] * coef[3 * s] : w[row + s * b];
    }
}

// Y(:, j, s) = X(:, j, s) for j < nlock[s]; then normalize every column of Y.
__global__ void restore_normalize_kernel(double* Y, const double* X, const int* nlock, int64_t r,
                                         int64_t b, const int* __restrict__ zmap) {
    const int64_t s = zmap ? (int64_t)zmap[blockIdx.y] : (int64_t)blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (j >= b) return;
    double* y = Y + (s * b + j) * r;
    if (j < nlock[s]) {
        const double* x = X + (s * b + j) * r;
        for (int64_t i = lane; i < r; i += 32) y[i] = x[i];
        return;
    }
    double acc = 0.0;
    for (int64_t i = lane; i < r; i += 32) acc = fma(y[i], y[i], acc);
    acc = warp_sum(acc);
    const double inv = acc > 0.0 ? rsqrt(acc) : 0.0;
    for (int64_t i = lane; i < r; i += 32) y[i] *= inv;
}

// res(j, s) = || GX(:, j, s) - theta(j, s) X(:, j, s) ||
__global__ void residual_kernel(const double* GX, const double* X, const double* theta,
                                double* res, int64_t r, int64_t b, const int* __restrict__ zmap) {
    const int64_t s = zmap ? (int64_t)zmap[blockIdx.y] : (int64_t)blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (j >= b) return;
    const double* g = GX + (s * b + j) * r;
    const double* x = X + (s * b + j) * r;
    const double th = theta[s * b + j];
    double acc = 0.0;
    for (int64_t i = lane; i < r; i += 32) {
        const double d = g[i] - th * x[i];
        acc = fma(d, d, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) res[s * b + j] = sqrt(acc);
}

// One CTA per slice: R = chol(S + shift*I) (upper, S = R^T R), then R^{-1},
// written out as a full b x b column-major block with zeros below the
// diagonal (Rout: R itself, optional; rows of non-positive pivots zeroed).
// b <= 160 (shared memory).
//
// The factor is built as L = R^T (lower, column-major in shared memory), so
// a row of R is a contiguous column of L. Right-looking, one barrier per
// step: step k updates the trailing lower triangle from the still unscaled
// column k and d = M(k,k) (M(i,j) -= M(i,k) M(j,k) / d) while column k-1 is
// scaled by 1/sqrt(d_{k-1}) (no longer read). R^{-1} is then solved column by
// column (R x = e_j), one warp per column: x lives in registers (lane l holds
// x(l + 32 t)), each back-substitution step is a lane-parallel dot with a
// fixed butterfly reduction.
constexpr int kCholSlots = 5;  // x slots per lane: b <= 160
__global__ void __launch_bounds__(1024, 1) chol_inv_kernel(const double* __restrict__ S, double* __restrict__ Rinv, int64_t b64,
                                int shift_pass, int* fail, double* __restrict__ Rout,
                                const int* __restrict__ zmap = nullptr, int* __restrict__ weak = nullptr) {
    extern __shared__ __align__(16) double M[];
    __shared__ double dinv[160];  // 1 / R(i,i)
    __shared__ unsigned char badk[160];  // pivot k broke down (a zero column)
    __shared__ int bad;
    const int b = (int)b64;
    const int64_t sl = zmap ? (int64_t)zmap[blockIdx.x] : (int64_t)blockIdx.x;
    const double* Sin = S + sl * b64 * b64;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (int i = tid; i < b * b; i += nt) M[i] = Sin[i];
    if (tid == 0) bad = 0;
    __syncthreads();
    if (shift_pass) {  // shifted CholQR (Fukaya et al.): tiny diagonal shift ~ u * trace
        double t = 0.0;
        for (int i = 0; i < b; ++i) t += M[i + i * b];  // every thread, same order
        __syncthreads();
        const double sh = 1e-15 * t;
        for (int i = tid; i < b; i += nt) M[i + i * b] += sh;
        __syncthreads();
    }
    if (b > 32 * kCholSlots) {  // the host sizes b <= 160 (shared memory)
        if (tid == 0 && fail) atomicExch(fail, 1);
        return;
    }
    // weak (nullable, one int per slice): set when a pivot falls below
    // 1e-12 of the largest diagonal, i.e. a column's residual after the
    // earlier ones is below 1e-6 of the largest column: CholQR's squared
    // condition number no longer yields an orthonormal factor there
    double dmax = 0.0;
    if (weak)
        for (int i = 0; i < b; ++i) dmax = fmax(dmax, M[i + i * b]);  // every thread, same order
    double dprev = 1.0;
    for (int k = 0; k < b; ++k) {
        const double d = M[k + k * b];
        const bool ok = d > 0.0;
        if (weak && tid == 0 && !(d > 1e-12 * dmax)) weak[sl] = 1;
        const double dk = ok ? d : 1.0;
        const double rinv = 1.0 / dk;
        // trailing lower triangle i >= j > k: warps over columns, lanes over rows
        for (int j = k + 1 + warp; j < b; j += nw) {
            const double mj = M[j + k * b] * rinv;
            for (int i = j + lane; i < b; i += 32) M[i + j * b] = fma(-M[i + k * b], mj, M[i + j * b]);
        }
        // column k-1 is final: scale it (rows > k-1) by 1/sqrt(d_{k-1})
        if (k > 0) {
            const double sc = 1.0 / sqrt(dprev);
            for (int i = k + tid; i < b; i += nt) M[i + (k - 1) * b] *= sc;
        }
        if (tid == 0) {
            if (!ok) bad = 1;
            badk[k] = !ok;
            dinv[k] = 1.0 / sqrt(dk);
        }
        dprev = dk;
        __syncthreads();
        if (tid == 0) M[k + k * b] = sqrt(dk);  // read by nobody after this step
    }
    __syncthreads();  // the last diagonal
    // now M holds L = R^T below the diagonal; R(i, l) = M[l + i*b] for l >= i
    if (Rout) {
        double* ro = Rout + sl * b64 * b64;
        for (int t = tid; t < b * b; t += nt) {
            const int i = t % b, jj = t / b;
            // a broken-down pivot's row of R is zero (W = Q R with W's column
            // in the span of the earlier ones, e.g. a zero slice): R^{-1} keeps
            // the unit pivot so Q stays finite
            ro[t] = (i <= jj && !badk[i]) ? M[jj + i * b] : 0.0;
        }
    }
    double* out = Rinv + sl * b64 * b64;
    // R x = e_j, x(i) = -(sum_{l=i+1..j} R(i,l) x(l)) / R(i,i); columns dealt to
    // the warps in a zig-zag so every warp gets a similar number of steps
    for (int c = warp; c < b; c += nw) {
        const int round = c / nw, pos = c % nw;
        const int cnt = b - round * nw < nw ? b - round * nw : nw;  // columns in this round
        const int j = (round & 1) ? (round * nw + (cnt - 1 - pos)) : c;
        double x[kCholSlots];
#pragma unroll
        for (int t = 0; t < kCholSlots; ++t) x[t] = 0.0;
        const double xj = dinv[j];
#pragma unroll
        for (int t = 0; t < kCholSlots; ++t)
            if (lane + 32 * t == j) x[t] = xj;
        for (int i = j - 1; i >= 0; --i) {
            const double* Li = M + i * b;  // row i of R: Li[l], l >= i
            double part = 0.0;
#pragma unroll
            for (int t = 0; t < kCholSlots; ++t) {
                const int l = lane + 32 * t;
                if (l > i && l <= j) part = fma(Li[l], x[t], part);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            const double xi = -part * dinv[i];
#pragma unroll
            for (int t = 0; t < kCholSlots; ++t)
                if (lane + 32 * t == i) x[t] = xi;
        }
        // column j of R^{-1}: rows 0..j from the lanes' slots, zeros below
#pragma unroll
        for (int t = 0; t < kCholSlots; ++t) {
            const int i = lane + 32 * t;
            if (i < b) out[i + (int64_t)j * b] = i <= j ? x[t] : 0.0;
        }
    }
    if (tid == 0 && bad && fail) atomicExch(fail, 1);
}

// Block-wide sum with a fixed order (warp butterflies, then warp 0 over the
// per-warp partials); every thread gets the result. red: >= 33 doubles.
__device__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();  // red is free (previous use finished)
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double a = lane < nw ? red[lane] : 0.0;
        a = warp_sum(a);
        if (lane == 0) red[32] = a;
    }
    __syncthreads();
    return red[32];
}

// The polish's QR of W (o x k per slice) for slices whose CholQR2 hit a weak
// pivot (rank-deficient slices, k above the slice rank, zero slices): CGS2
// (two classical Gram-Schmidt passes per column, which stays orthonormal to
// working precision at any condition number), one CTA per flagged slice.
// A column whose twice-projected residual is below 1e-14 of the largest
// column of W carries no content: it is replaced by an orthonormal
// completion, e_t projected out of the earlier columns with t the row of
// least captured mass (first on ties). Then R = Qw^T W (a general k x k; the
// Jacobi SVD of R that follows does not need it triangular), so W = Qw R
// holds to working precision and U = Qw Ur is orthonormal, as the
// reference's JacobiSVD factors are (matrix_kernels.cpp:29-37).
__global__ void __launch_bounds__(512) cgs2_fallback_kernel(const double* __restrict__ W, double* __restrict__ Qw,
                                                            double* __restrict__ R, int64_t o, int k,
                                                            const int* __restrict__ weak, double* __restrict__ dots) {
    const int64_t sl = blockIdx.x;
    if (!weak[sl]) return;
    __shared__ double red[33];
    __shared__ double c[160];
    __shared__ int tmin;
    const double* w = W + sl * o * k;
    double* q = Qw + sl * o * k;
    double* rowm = dots + sl * o;  // captured mass per row, sum_i q_i(t)^2
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    double wmax = 0.0;
    for (int j = 0; j < k; ++j) {
        double a = 0.0;
        for (int64_t t = tid; t < o; t += nt) a = fma(w[t + j * o], w[t + j * o], a);
        wmax = fmax(wmax, block_sum(a, red));
    }
    for (int64_t t = tid; t < o; t += nt) rowm[t] = 0.0;
    for (int j = 0; j < k; ++j) {
        double* v = q + (int64_t)j * o;
        for (int64_t t = tid; t < o; t += nt) v[t] = w[t + (int64_t)j * o];
        double nv = 0.0;
        for (int attempt = 0; attempt < 2; ++attempt) {
            for (int pass = 0; pass < 2; ++pass) {
                __syncthreads();
                // c_i = q_i^T v (one warp per i, lanes over rows, fixed order)
                for (int i = warp; i < j; i += nw) {
                    const double* qi = q + (int64_t)i * o;
                    double a = 0.0;
                    for (int64_t t = lane; t < o; t += 32) a = fma(qi[t], v[t], a);
                    a = warp_sum(a);
                    if (lane == 0) c[i] = a;
                }
                __syncthreads();
                for (int64_t t = tid; t < o; t += nt) {
                    double x = v[t];
                    for (int i = 0; i < j; ++i) x = fma(-q[t + (int64_t)i * o], c[i], x);
                    v[t] = x;
                }
            }
            double a = 0.0;
            for (int64_t t = tid; t < o; t += nt) a = fma(v[t], v[t], a);
            nv = block_sum(a, red);
            if (attempt == 1 || nv > 1e-28 * wmax) break;
            // no content left: start over from e_t, t = the least captured row
            if (tid == 0) {
                int64_t best = 0;
                for (int64_t t = 1; t < o; ++t)
                    if (rowm[t] < rowm[best]) best = t;
                tmin = (int)best;
            }
            __syncthreads();
            for (int64_t t = tid; t < o; t += nt) v[t] = t == tmin ? 1.0 : 0.0;
        }
        const double inv = nv > 0.0 ? 1.0 / sqrt(nv) : 0.0;
        for (int64_t t = tid; t < o; t += nt) {
            const double x = v[t] * inv;
            v[t] = x;
            rowm[t] = fma(x, x, rowm[t]);
        }
    }
    __syncthreads();
    // R = Qw^T W: one warp per entry
    double* r = R + sl * (int64_t)k * k;
    for (int e = warp; e < k * k; e += nw) {
        const int i = e % k, jj = e / k;
        const double* qi = q + (int64_t)i * o;
        const double* wj = w + (int64_t)jj * o;
        double a = 0.0;
        for (int64_t t = lane; t < o; t += 32) a = fma(qi[t], wj[t], a);
        a = warp_sum(a);
        if (lane == 0) r[e] = a;
    }
}

// tail2[z] = sum of the pairs' first components of CTA partials in group z.
__global__ void group_sum_kernel(const double* part, int64_t per_group, double* out) {
    const int64_t z = blockIdx.x;
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < per_group; i += blockDim.x) a += part[2 * (z * per_group + i)];
    __shared__ double red[32];
    a = warp_sum(a);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
        a = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        a = warp_sum(a);
        if (threadIdx.x == 0) out[z] = a;
    }
}

// out[s] = max_i G_s(i, i): for a PSD G every |G(i, j)| <= sqrt(G_ii G_jj) is
// bounded by it, so it scales all columns of the slice alike (symmetric split).
__global__ void diag_max_kernel(const double* __restrict__ G, int64_t r, double* __restrict__ out) {
    const double* g = G + (int64_t)blockIdx.x * r * r;
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < r; i += blockDim.x) m = fmax(m, fabs(g[i + i * r]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
        out[blockIdx.x] = fmax(m, red[0]);
    }
}

// th(c0 + j, s) = P(j, s), j < bc, for the slices of the launch (zmap).
__global__ void copy_theta_kernel(double* __restrict__ th, const double* __restrict__ P, int64_t b,
                                  int64_t bc, int64_t c0, const int* __restrict__ zmap) {
    const int64_t s = zmap ? (int64_t)zmap[blockIdx.x] : (int64_t)blockIdx.x;
    for (int64_t j = threadIdx.x; j < bc; j += blockDim.x) th[s * b + c0 + j] = P[s * bc + j];
}

// Slices that stopped filtering before the last degree left their block in
// another buffer of the (Yp, Y, Yn) rotation: dst(:, s) = src[from[z]](:, s).
__global__ void gather_filtered_kernel(double* __restrict__ dst, const double* __restrict__ b0,
                                       const double* __restrict__ b1, const double* __restrict__ b2,
                                       const int* __restrict__ list, int64_t per) {
    const int s = list[2 * blockIdx.y], from = list[2 * blockIdx.y + 1];
    const double* src = from == 0 ? b0 : (from == 1 ? b1 : b2);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x)
        dst[s * per + i] = src[s * per + i];
}

unsigned grid1(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

// ---------------------------------------------------------------- GEMM glue
// C_s (rows x cols) = alpha * X_s^T (rows x m)^T ... helpers for the batched
// r x b panels (column-major, per-slice strides).
void g_AtB(const double* A, const double* B, double* C, int64_t m, int64_t ra, int64_t rb,
           int64_t batch, int64_t sA, int64_t sB, cudaStream_t s, const int* zmap = nullptr,
           int64_t zext = 0) {
    // C (ra x rb) = A^T (ra x m) * B (m x rb); A is m x ra, B is m x rb
    GemmDesc d;
    d.zmap = zmap;
    d.zmap_extent = zext;
    d.M = ra; d.N = rb; d.K = m; d.batch = batch;
    d.A = A; d.lda = m; d.strideA = sA; d.a_kmajor = true;
    d.B = B; d.ldb = m; d.strideB = sB;
    d.C = C; d.ldc = ra; d.strideC = ra * rb;
    gemm(d, s);
}

void g_AB(const double* A, const double* B, double* C, int64_t m, int64_t kk, int64_t n,
          int64_t batch, int64_t sA, int64_t sB, double alpha, const double* Cin, double beta,
          cudaStream_t s, const int* zmap = nullptr, int64_t zext = 0) {
    // C (m x n) = alpha * A (m x kk) * B (kk x n) + beta * Cin
    GemmDesc d;
    d.zmap = zmap;
    d.zmap_extent = zext;
    d.M = m; d.N = n; d.K = kk; d.batch = batch;
    d.A = A; d.lda = m; d.strideA = sA;
    d.B = B; d.ldb = kk; d.strideB = sB;
    d.C = C; d.ldc = m; d.strideC = m * n;
    d.alpha = alpha;
    d.Cin = Cin; d.ldcin = m; d.strideCin = m * n; d.beta = beta;
    gemm(d, s);
}

struct Work {
    int64_t r, b, batch;
    bool basis = false;  // eigenbasis Q (data_q) rather than slice SVDs: stage names sq.*
    DeviceBuffer X, Y, Yp, Yn, Z, W, P, S, Rinv, Hv, th, res, coef, wmask, nlock, fail, zmap, glist, Ssplit;
    Work(int64_t r_, int64_t b_, int64_t batch_)
        : r(r_), b(b_), batch(batch_),
          X(sizeof(double) * r_ * b_ * batch_), Y(sizeof(double) * r_ * b_ * batch_),
          Yp(sizeof(double) * r_ * b_ * batch_), Yn(sizeof(double) * r_ * b_ * batch_),
          Z(sizeof(double) * r_ * b_ * batch_), W(sizeof(double) * r_ * b_ * batch_),
          P(sizeof(double) * b_ * b_ * batch_), S(sizeof(double) * b_ * b_ * batch_),
          Rinv(sizeof(double) * b_ * b_ * batch_), Hv(sizeof(double) * b_ * b_ * batch_),
          th(sizeof(double) * b_ * batch_), res(sizeof(double) * b_ * batch_),
          coef(sizeof(double) * 3 * batch_), wmask(sizeof(double) * b_ * batch_),
          nlock(sizeof(int) * batch_), fail(sizeof(int) * 2), zmap(sizeof(int) * batch_),
          Ssplit(panel_kernels_ok(r_, std::min<int64_t>(b_, 64))
                     ? sizeof(double) * b_ * b_ * batch_ * panel_splits(r_)
                     : 0) {}
};

// General strided-batch GEMM on column panels: C = alpha op(A) B + beta C.
void gg(const double* A, int64_t lda, int64_t sA, bool at, const double* B, int64_t ldb, int64_t sB,
        double* C, int64_t ldc, int64_t sC, int64_t M, int64_t N, int64_t K, int64_t batch,
        double alpha, double beta, cudaStream_t s, const int* zmap = nullptr, int64_t zext = 0) {
    GemmDesc d;
    d.M = M; d.N = N; d.K = K; d.batch = batch; d.zmap = zmap; d.zmap_extent = zext;
    d.A = A; d.lda = lda; d.strideA = sA; d.a_kmajor = at;
    d.B = B; d.ldb = ldb; d.strideB = sB;
    d.C = C; d.ldc = ldc; d.strideC = sC;
    d.alpha = alpha;
    if (beta != 0.0) { d.Cin = C; d.ldcin = ldc; d.strideCin = sC; d.beta = beta; }
    gemm(d, s);
}

// Orthonormalize columns [c0, b) of the r x b panels Y into the same columns
// of Xout: first against the locked columns [0, c0) of X (block CGS, twice),
// then shifted CholQR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa
// 2020): the shifted first pass keeps the Cholesky factorization alive for
// cond(Y) up to ~1e15, two plain passes restore orthogonality.
void cholqr3(Work& w, double* Y, double* Xout, int64_t c0, cudaStream_t s, const int* zm = nullptr,
             int64_t na = -1) {
    HostProf hp_("cholqr3");
    const int64_t r = w.r, b = w.b, bc = b - c0, per = r * b;
    const int64_t batch = na < 0 ? w.batch : na;  // launched slices (zm: which ones)
    const int64_t zx = w.batch;
    StageTimer tm(w.basis ? "sq.cholqr3" : "ss.cholqr3", s);
    if (c0 > 0)
        for (int pass = 0; pass < 2; ++pass) {
            // P = X_L^T Y_A (c0 x bc); Y_A -= X_L P
            gg(w.X.d(), r, per, true, Y + c0 * r, r, per, w.P.d(), c0, c0 * bc, c0, bc, r, batch, 1.0, 0.0, s, zm, zx);
            gg(w.X.d(), r, per, false, w.P.d(), c0, c0 * bc, Y + c0 * r, r, per, r, bc, c0, batch, -1.0, 1.0, s, zm,
               zx);
        }
    const size_t smem = (size_t)bc * bc * sizeof(double);
    if (smem > 200 * 1024) fail(PPC_ARGUMENT, "subspace: block too wide for the CholQR kernel");
    if (smem > 48 * 1024)
        PPC_CUDA_CHECK(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem));
    double* src = Y + c0 * r;
    double* bufs[3] = {w.Yn.d() + c0 * r, w.Z.d() + c0 * r, Xout + c0 * r};
    const bool small = panel_kernels_ok(r, bc);
    for (int pass = 0; pass < 3; ++pass) {
        if (small) {
            // S = Y^T Y (split-K partials summed in split order, panel.cu)
            panel_gram(src, per, src, per, r, bc, batch, w.S.d(), w.Ssplit.d(), zx, zm, s);
            chol_inv64(w.S.d(), bc, batch, pass == 0, w.Rinv.d(), w.fail.as<int>(), zm, nullptr, s);
            panel_apply(src, per, w.Rinv.d(), bufs[pass], per, r, bc, batch, zm, s);
        } else {
            gg(src, r, per, true, src, r, per, w.S.d(), bc, bc * bc, bc, bc, r, batch, 1.0, 0.0, s, zm, zx);
            chol_inv_kernel<<<(unsigned)batch, bc > 16 ? 1024 : 256, smem, s>>>(
                w.S.d(), w.Rinv.d(), bc, pass == 0 ? 1 : 0, w.fail.as<int>(), nullptr, zm);
            count_launch();
            check_launch("chol_inv");
            gg(src, r, per, false, w.Rinv.d(), bc, bc * bc, bufs[pass], r, per, r, bc, bc, batch, 1.0, 0.0, s, zm,
               zx);
        }
        src = bufs[pass];
    }
}

}  // namespace

// Shifted CholQR3 of one r x k panel in place (the direct eigensolver's
// inverse-iteration vectors): column order is kept, so Z R^{-1} is a
// Gram-Schmidt of Z in eigenvalue order.
void cholqr_inplace(double* Z, int64_t r, int64_t k, cudaStream_t s, int64_t batch) {
    if (k > 160) fail(PPC_ARGUMENT, "cholqr_inplace: too many columns");
    DeviceBuffer S(sizeof(double) * k * k * batch), Ri(sizeof(double) * k * k * batch),
        T(sizeof(double) * r * k * batch);
    const size_t smem = (size_t)k * k * sizeof(double);
    if (smem > 48 * 1024)
        PPC_CUDA_CHECK(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem));
    double* src = Z;
    double* dst = T.d();
    for (int pass = 0; pass < 3; ++pass) {
        gg(src, r, r * k, true, src, r, r * k, S.d(), k, k * k, k, k, r, batch, 1.0, 0.0, s);  // S = Z^T Z
        chol_inv_kernel<<<(unsigned)batch, k > 16 ? 1024 : 256, smem, s>>>(S.d(), Ri.d(), k, pass == 0 ? 1 : 0,
                                                                          nullptr, nullptr);
        count_launch();
        check_launch("chol_inv");
        gg(src, r, r * k, false, Ri.d(), k, k * k, dst, r, r * k, r, k, k, batch, 1.0, 0.0, s);
        std::swap(src, dst);
    }
    if (src != Z)
        PPC_CUDA_CHECK(cudaMemcpyAsync(Z, src, sizeof(double) * r * k * batch, cudaMemcpyDeviceToDevice, s));
}

namespace {

// Rayleigh-Ritz on the orthonormal active columns [c0, b) of Xn: X, theta,
// W = G X and residual norms for those columns (locked ones keep theirs).
// Gd (nullable): G's Ozaki digits; then Z = G Xn runs on the INT8 tensor
// cores at full digit depth (~1e-14 |G|, far below every residual the
// caller still acts on; it passes nullptr near the lock thresholds).
void rayleigh_ritz(Work& w, const double* G, int64_t sG, double* Xn, int64_t c0, cudaStream_t s,
                   double gtol_rel, int sweep_cap, const int* zm = nullptr, int64_t na = -1,
                   const OzakiDigits* Gd = nullptr, OzakiDigits* Xd = nullptr) {
    HostProf hp_("rayleigh_ritz");
    const int64_t r = w.r, b = w.b, bc = b - c0, per = r * b;
    const int64_t batch = na < 0 ? w.batch : na;  // launched slices (zm: which ones)
    const int64_t zx = w.batch;
    StageTimer tm(w.basis ? "sq.rayleigh_ritz" : "ss.rayleigh_ritz", s);
    if (Gd && Xd && bc <= 64) {
        Xd->split(Xn + c0 * r, r, per, r, bc, r, zx, s, zm, zm ? batch : 0);
        if (zm) {
            ozaki_gemm(*Gd, *Xd, batch, zm, w.Z.d() + c0 * r, r, per, s, 6, true);
        } else {
            ozaki_gemm(*Gd, *Xd, batch, nullptr, w.Z.d() + c0 * r, r, per, s, 6, true);
        }
    } else {
        gg(G, r, sG, false, Xn + c0 * r, r, per, w.Z.d() + c0 * r, r, per, r, bc, r, batch, 1.0, 0.0, s, zm,
           zx);  // Z = G Xn
    }
    const bool small = panel_kernels_ok(r, bc);
    if (small) {  // H = Xn^T Z (= Xn^T G Xn): upper triangle, mirrored
        panel_gram(Xn + c0 * r, per, w.Z.d() + c0 * r, per, r, bc, batch, w.S.d(), w.Ssplit.d(), zx, zm, s);
    } else {
        gg(Xn + c0 * r, r, per, true, w.Z.d() + c0 * r, r, per, w.S.d(), bc, bc * bc, bc, bc, r, batch, 1.0, 0.0, s,
           zm, zx);
    }
    {
        StageTimer tj(w.basis ? "sq.rr_eig" : "ss.rr_eig", s);
        // H (PSD) = Hv diag(theta) Hv^T by one-sided Jacobi (eigen mode)
        jacobi_svd(w.S.d(), bc, bc, bc * bc, batch, bc, nullptr, w.P.d(), w.Hv.d(), nullptr, s, gtol_rel,
                   sweep_cap, zm);
    }
    copy_theta_kernel<<<(unsigned)batch, 64, 0, s>>>(w.th.d(), w.P.d(), b, bc, c0, zm);
    count_launch();
    check_launch("copy_theta");
    if (small) {
        panel_apply(Xn + c0 * r, per, w.Hv.d(), w.X.d() + c0 * r, per, r, bc, batch, zm, s);
        panel_apply(w.Z.d() + c0 * r, per, w.Hv.d(), w.W.d() + c0 * r, per, r, bc, batch, zm, s);
    } else {
        gg(Xn + c0 * r, r, per, false, w.Hv.d(), bc, bc * bc, w.X.d() + c0 * r, r, per, r, bc, bc, batch, 1.0, 0.0,
           s, zm, zx);
        gg(w.Z.d() + c0 * r, r, per, false, w.Hv.d(), bc, bc * bc, w.W.d() + c0 * r, r, per, r, bc, bc, batch, 1.0,
           0.0, s, zm, zx);
    }
    dim3 grid((unsigned)((b + 7) / 8), (unsigned)batch);
    residual_kernel<<<grid, 256, 0, s>>>(w.W.d(), w.X.d(), w.th.d(), w.res.d(), r, b, zm);
    count_launch();
    check_launch("residual");
}

}  // namespace

// Reduced-precision filter products while every unlocked residual of a slice
// exceeds this fraction of its theta_1 (PPC_FILTER_LOWP; 0 disables): 4 digit
// levels above it, 3 levels above 1000x it.
static double filter_lowp() {
    static const double v = std::getenv("PPC_FILTER_LOWP") ? std::atof(std::getenv("PPC_FILTER_LOWP")) : 1e-6;
    return v;
}

// Chebyshev degree cap per outer iteration (runtime-tunable for experiments).
// 20 with the INT8 reduced-level filter, where a degree costs less than the
// CholQR3 + Rayleigh-Ritz of an extra outer iteration (cfg5 slice SVD 56 ->
// 50 ms); 10 with the FP64 filter of small slices (cfg3: 20 is 12% slower).
static double max_degree(bool basis, bool int8_filter) {
    static const char* e = std::getenv("PPC_CHEB_MAX");
    static const double v = e ? std::atof(e) : 0.0;
    static const double vq = std::getenv("PPC_CHEB_MAX_Q") ? std::atof(std::getenv("PPC_CHEB_MAX_Q")) : 10.0;
    if (basis) return vq;
    return v > 0.0 ? v : (int8_filter ? 20.0 : 10.0);
}

// tail2[z] = ||A_z - U_z diag(S_z) V_z^T||_F^2 (= the discarded energy sum_{j>=k} s_j^2
// of slice z by Eckart-Young), via the fused residual GEMM.
void slice_tail_energy(const double* A, int64_t m, int64_t n, int64_t stride, int64_t batch,
                       int64_t k, const double* U, const double* S, const double* V, double* tail2,
                       cudaStream_t s) {
    DeviceBuffer us(sizeof(double) * m * k * batch);
    launch_scale_columns(U, S, us.d(), m, k, batch, s);
    GemmDesc d;
    d.M = m; d.N = n; d.K = k; d.batch = batch;
    d.A = us.d(); d.lda = m; d.strideA = m * k;
    d.B = V; d.ldb = n; d.strideB = n * k; d.b_nmajor = true;
    d.allow_ws = false;  // per-batch CTA groups are needed for the per-slice sums
    const int64_t ctas = gemm_residual_ctas(d, A, m, stride);
    DeviceBuffer part(sizeof(double) * 2 * ctas);
    gemm_residual(d, A, m, stride, part.d(), s);
    group_sum_kernel<<<(unsigned)batch, 256, 0, s>>>(part.d(), ctas / batch, tail2);
    count_launch();
    check_launch("group_sum");
}

// Top-k eigenpairs of `batch` symmetric PSD r x r matrices G (stride r*r).
// Xout (r, k, batch), lambda (k, batch). Deterministic.
void subspace_eig_top(const double* G, int64_t r, int64_t batch, int64_t k, double* Xout,
                      double* lambda, cudaStream_t s, bool vectors_for_reconstruction) {
    HostProf hp_("subspace_eig_top");
    static const bool dbg = std::getenv("PPC_SUBSPACE_DEBUG") != nullptr;
    static const int64_t guard_env = std::getenv("PPC_SUBSPACE_GUARD") ? std::atoll(std::getenv("PPC_SUBSPACE_GUARD")) : 0;
    int64_t b = k + (guard_env > 0 ? guard_env : std::max<int64_t>(k, 16));
    b = (b + 7) / 8 * 8;
    if (b >= r || r <= 8) {
        // the block would cover the space: full Jacobi eigendecomposition
        jacobi_svd(G, r, r, r * r, batch, k, nullptr, lambda, Xout, nullptr, s);
        return;
    }
    b = std::min<int64_t>(b, 160);
    if (k > b) fail(PPC_ARGUMENT, "subspace_eig_top: k too large for the block");
    Work w(r, b, batch);
    w.basis = !vectors_for_reconstruction;
    const int64_t per = r * b;
    // Chebyshev filter products G Y on the INT8 tensor cores (Ozaki, 7
    // digits): G is split once, the block Y at every degree. Rayleigh-Ritz
    // and the residuals keep the FP64 DMMA products, so locking and the
    // final accuracy do not depend on the emulated filter.
    // below r = 1024 the per-degree digit splits and short persistent launches
    // cost more than the FP64 DMMA products they replace (cfg3: 13.8 -> 12.8 ms)
    static const int64_t oz_min_r =
        std::getenv("PPC_OZ_FILTER_MIN_R") ? std::atoll(std::getenv("PPC_OZ_FILTER_MIN_R")) : 1024;
    const bool oz_filter = vectors_for_reconstruction && batch >= 8 && r >= oz_min_r && ozaki_gemm_eligible(r, r);
    OzakiDigits Gd, Yd;
    DeviceBuffer gmax;
    if (oz_filter) {
        // one scale per slice Gram (bounded by its largest diagonal entry): the
        // filter and Rayleigh-Ritz products then read G from its upper triangle
        gmax = DeviceBuffer(sizeof(double) * batch);
        diag_max_kernel<<<(unsigned)batch, 256, 0, s>>>(G, r, gmax.d());
        count_launch();
        check_launch("diag_max");
        Gd.split(G, r, r * r, r, r, r, batch, s, nullptr, 0, 0, 0, nullptr, 6, 0, 0, gmax.d());
    }
    PPC_CUDA_CHECK(cudaMemsetAsync(w.fail.d(), 0, 2 * sizeof(int), s));
    randn_kernel<<<grid1(per * batch), 256, 0, s>>>(w.Y.d(), per * batch, 0x5eed5eedULL + (uint64_t)r * 131 + b);
    count_launch();
    cholqr3(w, w.Y.d(), w.Yp.d(), 0, s);
    const double gtol_rel = vectors_for_reconstruction ? 0.0 : 1e-14;
    // early Rayleigh-Ritz steps only steer the filter: 4 Jacobi sweeps
    rayleigh_ritz(w, G, r * r, w.Yp.d(), 0, s, gtol_rel, 4, nullptr, -1, oz_filter ? &Gd : nullptr, &Yd);

    std::vector<double> th(b * batch), res(b * batch), coef(3 * batch), wm(b * batch),
        thp(b * batch, 0.0);
    std::vector<int> nlock(batch, 0);
    // reduced-level filter guard: a slice whose smallest unlocked residual
    // stopped halving between iterations while filtered at reduced precision
    // is held at the next precision level from then on (cap[sl])
    std::vector<double> prev_rmin(batch, 1e300);
    std::vector<char> cap(batch, 2);
    const int max_iter = 100;
    auto tprev = std::chrono::steady_clock::now();
    for (int it = 0; it < max_iter; ++it) {
        PPC_CUDA_CHECK(cudaMemcpyAsync(th.data(), w.th.d(), sizeof(double) * b * batch, cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaMemcpyAsync(res.data(), w.res.d(), sizeof(double) * b * batch, cudaMemcpyDeviceToHost, s));
        const auto tq = std::chrono::steady_clock::now();
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
        if (dbg) {  // host time of the last iteration (the pageable D2H above already waited for the GPU)
            const auto tw = std::chrono::steady_clock::now();
            fprintf(stderr, "[subspace] it %d host enqueue %.3f ms, wait %.3f ms\n", it,
                    std::chrono::duration<double, std::milli>(tq - tprev).count(),
                    std::chrono::duration<double, std::milli>(tw - tq).count());
            tprev = tw;
        }
        bool all_done = true;
        int dmax = 0;
        // ||A||^2 ~ sum of the slices' captured energies (top-b Ritz values)
        double energy = 0.0;
        for (int64_t i = 0; i < b * batch; ++i) energy += std::max(th[i], 0.0);
        std::vector<int> deg(batch, 0);
        bool near_floor = false;
        // slices whose unlocked residuals are still far above the reduced
        // filter's precision floor (~1e-9 |G|): their products take 4 digit
        // levels (half the MMAs); locking always uses FP64 Rayleigh-Ritz
        // residuals, so this only steers the iteration
        std::vector<char> lowp(batch, 0);  // 0: 6 levels, 1: 4 levels, 2: 3 levels
        std::vector<double> cc(batch), ee(batch);
        for (int64_t sl = 0; sl < batch; ++sl) {
            const double* t = &th[sl * b];
            const double* rr = &res[sl * b];
            const double scale = std::max(t[0], 1e-300);
            // Lock a converged prefix. Singular values after the Rayleigh-Ritz
            // polish carry relative error ~ (res/gap)^2, so res <= 1e-9 theta_1
            // suffices for them. Slice-SVD vectors must also reproduce the
            // rank-k truncation to 1e-11 ||A||: the subspace angle is
            // res / (theta_k - theta_{k+1}), which moves A_k by about
            // angle * (sigma_k + sigma_{k+1}). The eigenbasis Q only needs
            // eigenvalue accuracy (res <= 1e-13 theta_1).
            double thr;
            if (vectors_for_reconstruction) {
                const double gap = std::max(t[k - 1] - t[k], 0.0);
                const double srec = 1e-11 * std::sqrt(energy) * gap /
                                    (std::sqrt(std::max(t[k - 1], 0.0)) + std::sqrt(std::max(t[k], 0.0)) + 1e-300);
                // polished singular values err by ~ sigma_j * angle^2, angle ~ res/gap
                const double ssig = 3e-6 * gap;
                thr = std::max(32.0 * 2.22e-16 * scale, std::min(srec, ssig));
            } else {
                thr = 1e-13 * scale;
            }
            int L = 0;
            std::vector<double> thrv(k, thr);
            if (vectors_for_reconstruction && it >= 2) {
                // Per-column thresholds from Rayleigh-Ritz perturbation theory
                // on the b-column block (the k-boundary gap alone is far too
                // pessimistic on noise plateaus, where it is ~1e-3 theta_1):
                //  g_j   = gap from theta_j to the uncaptured spectrum, taken
                //          as half of theta_j - theta_b (theta_b <= lambda_b);
                //  (i)   Ritz value error <= ||R||^2 / g_j, and the polished
                //        sigma_j = sqrt(theta_j): res_j sqrt(k) <= sqrt(2e-10 theta_j g_j);
                //  (ii)  the kept subspace misses v_j by res_j / g_j, which moves
                //        the rank-k truncation by ~ sqrt(2) sigma_j res_j / g_j
                //        <= 1e-11 ||A||;
                //  (iii) x_j mixes with the discarded Ritz vectors by a further
                //        factor ||R|| / (theta_j - theta_k) (Saad, Thm 4.6).
                const double tout = std::max(t[b - 1], 0.0);
                double R2 = 0.0;
                for (int64_t j = 0; j < b; ++j) R2 += rr[j] * rr[j];
                const double Rn = std::sqrt(R2), sk = std::sqrt((double)k), sE = std::sqrt(energy);
                for (int64_t j = 0; j < k; ++j) {
                    const double tj = std::max(t[j], 0.0);
                    const double g = 0.5 * (tj - tout);
                    if (!(g > 0.0)) break;  // no separation from the block bottom: keep thr
                    const double sj = std::sqrt(tj);
                    const double ti = std::sqrt(2e-10 * tj * g) / sk;
                    const double cross = std::max(tj - t[k], 0.0);
                    const double tii = 1e-11 * sE * g / (1.4142135623730951 * sj + 1e-300) *
                                       std::min(1.0, cross / (Rn + 1e-300));
                    thrv[j] = std::max(thr, std::max(32.0 * 2.22e-16 * scale, std::min(ti, tii)));
                }
                // A locked column's residual couples into the deflated operator
                // and floors the residuals of the columns after it, so no column
                // may lock looser than any later wanted column needs.
                for (int64_t j = k - 2; j >= 0; --j) thrv[j] = std::min(thrv[j], thrv[j + 1]);
                while (L < k && rr[L] <= thrv[L]) ++L;
            } else if (vectors_for_reconstruction) {
                while (L < k && rr[L] <= thr) ++L;  // locked prefix
            } else {
                // basis Q: judged on eigenvalues / captured energy (SURVEY 8c
                // rule 5) -> also lock Ritz values that moved < 5e-13 theta_1
                // in the last iteration (linear convergence, rate ~0.35 on the
                // cfg5 noise plateau: remaining error ~0.5x the last move,
                // under the 1e-12 theta_1 parity bound)
                while (L < k && (rr[L] <= thr ||
                                 (it >= 2 && std::fabs(t[L] - thp[sl * b + L]) <= 5e-13 * scale &&
                                  rr[L] <= 1e-6 * scale)))
                    ++L;
            }
            nlock[sl] = L;
            for (int64_t j = 0; j < b; ++j) wm[sl * b + j] = (j < L) ? t[j] : 0.0;
            if (L >= k || t[0] <= 0.0) {
                deg[sl] = 0;
                continue;
            }
            all_done = false;
            // within ~1e-11 theta_1 of the lock thresholds the INT8 filter's
            // own rounding (~1e-14 |G| |Y|) would floor the residuals: filter
            // in FP64 from here on
            for (int64_t j = L; j < k; ++j)
                if (rr[j] <= 1e-11 * scale) near_floor = true;
            if (vectors_for_reconstruction && filter_lowp() > 0.0) {
                double rmin = 1e300;
                for (int64_t j = L; j < k; ++j) rmin = std::min(rmin, rr[j]);
                char lv = rmin > filter_lowp() * scale ? (rmin > 1e3 * filter_lowp() * scale ? 2 : 1) : 0;
                if (lv > 0 && lv == cap[sl] && it >= 2 && rmin > 0.5 * prev_rmin[sl]) cap[sl] = (char)(lv - 1);
                lowp[sl] = std::min(lv, cap[sl]);
                prev_rmin[sl] = rmin;
            }
            // Chebyshev interval [0, ub]: damp everything below the smallest Ritz value
            // (moving the bound up by the last column's residual, to cover the
            // eigenvalues just outside a block whose last Ritz value still lags,
            // measured much slower at cfg5: 142-149 ms a step against 118)
            const double ub = std::max(t[b - 1], 0.0);
            const double c = 0.5 * ub, e = std::max(0.5 * ub, 1e-300 * scale);
            cc[sl] = c;
            ee[sl] = e;
            const double xt = std::max(1.0, (t[L] - c) / e), xk = std::max(1.0, (t[k - 1] - c) / e);
            // (a) the block must stay numerically full rank for shifted
            // CholQR3: amplification of the largest active Ritz value over the
            // block's bottom (x = 1, T_d(1) = 1) kept <= 1e10;
            // (b) the spread inside the wanted active set (precision of the
            // smaller wanted components) kept <= 1e6.
            double d = max_degree(w.basis, oz_filter);
            if (xt > 1.0) d = std::min(d, std::acosh(1e10) / std::acosh(xt));
            const double spread = std::acosh(xt) - std::acosh(xk);
            if (spread > 0) d = std::min(d, std::log(1e6) / spread);
            if (xk <= 1.0 + 1e-12) d = std::min(d, 2.0);  // no separation yet: gentle
            // no more than this slice needs: the residuals of the unlocked
            // wanted columns fall by ~exp(-acosh(x_k)) per degree
            if (xk > 1.0 + 1e-12 && it >= 2) {
                double rmax = 1.0;  // largest residual / threshold ratio among unlocked wanted columns
                for (int64_t j = L; j < k; ++j) rmax = std::max(rmax, rr[j] / thrv[j]);
                // (1.4x and two spare degrees: the asymptotic rate overestimates the
                // first degrees after a restart, and a cleanup iteration for a
                // handful of columns costs a whole CholQR3 + Rayleigh-Ritz round;
                // cfg5: 6 -> 5 rounds, slice SVD 44.7 -> 43.0 ms)
                const double need = std::log(rmax) / std::acosh(xk);
                static const double need_scale = std::getenv("PPC_NEED_SCALE") ? std::atof(std::getenv("PPC_NEED_SCALE")) : 1.4;
                static const double need_add = std::getenv("PPC_NEED_ADD") ? std::atof(std::getenv("PPC_NEED_ADD")) : 2.0;
                d = std::min(d, std::max(1.0, std::ceil(need_scale * need) + need_add));
            }
            deg[sl] = std::max(1, (int)d);
            dmax = std::max(dmax, deg[sl]);
            if (dbg && (sl < 4 || it % 10 == 0))
                fprintf(stderr, "[subspace] it %d slice %lld L=%d deg=%d t0=%.6e tk=%.6e tb=%.6e res0=%.3e resk=%.3e thr=%.3e\n",
                        it, (long long)sl, L, deg[sl], t[0], t[k - 1], t[b - 1], rr[0], rr[k - 1], thr);
        }
        if (dbg) {
            int nact_sl = 0;
            std::string act;
            for (int64_t sl = 0; sl < batch; ++sl)
                if (deg[sl] > 0) {
                    ++nact_sl;
                    if (act.size() < 600)
                        act += " " + std::to_string(sl) + ":" + std::to_string(nlock[sl]) + "/" + std::to_string(deg[sl]);
                }
            fprintf(stderr, "[subspace] it %d dmax %d active %d (slice:L/deg)%s\n", it, dmax, nact_sl, act.c_str());
        }
        thp = th;
        if (all_done) break;
        PPC_CUDA_CHECK(cudaMemcpyAsync(w.wmask.d(), wm.data(), sizeof(double) * b * batch, cudaMemcpyHostToDevice, s));
        PPC_CUDA_CHECK(cudaMemcpyAsync(w.nlock.d(), nlock.data(), sizeof(int) * batch, cudaMemcpyHostToDevice, s));
        // per-degree, per-slice recurrence coefficients (one upload per iteration)
        coef.assign(3 * batch * dmax, 0.0);
        for (int j = 0; j < dmax; ++j)
            for (int64_t sl = 0; sl < batch; ++sl) {
                double* cf = &coef[3 * (j * batch + sl)];
                if (j >= deg[sl]) {
                    cf[0] = 0.0; cf[1] = 1.0; cf[2] = 0.0;  // frozen: Y_{j+1} = Y_j
                } else if (j == 0) {
                    cf[0] = 1.0 / ee[sl]; cf[1] = -cc[sl] / ee[sl]; cf[2] = 0.0;
                } else {
                    cf[0] = 2.0 / ee[sl]; cf[1] = -2.0 * cc[sl] / ee[sl]; cf[2] = -1.0;
                }
            }
        if ((int64_t)coef.size() * 8 > (int64_t)w.coef.bytes()) w.coef = DeviceBuffer(coef.size() * sizeof(double));
        // per degree: every filtering slice | the reduced-precision ones | the rest
        std::vector<int> zm((size_t)4 * dmax * batch), nact(dmax, 0), nlo(dmax, 0), nhi(dmax, 0), nl3(dmax, 0);
        for (int j = 0; j < dmax; ++j)
            for (int64_t sl = 0; sl < batch; ++sl)
                if (j < deg[sl]) {
                    zm[(size_t)j * batch + nact[j]++] = (int)sl;
                    if (lowp[sl] == 1) zm[(size_t)(dmax + j) * batch + nlo[j]++] = (int)sl;
                    else if (lowp[sl] == 2) zm[(size_t)(3 * dmax + j) * batch + nl3[j]++] = (int)sl;
                    else zm[(size_t)(2 * dmax + j) * batch + nhi[j]++] = (int)sl;
                }
        if ((int64_t)zm.size() * 4 > (int64_t)w.zmap.bytes()) w.zmap = DeviceBuffer(zm.size() * sizeof(int));
        PPC_CUDA_CHECK(cudaMemcpyAsync(w.zmap.d(), zm.data(), sizeof(int) * zm.size(), cudaMemcpyHostToDevice, s));
        PPC_CUDA_CHECK(cudaMemcpyAsync(w.coef.d(), coef.data(), sizeof(double) * coef.size(), cudaMemcpyHostToDevice, s));
        // filter: Y_0 = X; Y_{j+1} from the deflated operator G - X_L Theta_L X_L^T
        PPC_CUDA_CHECK(cudaMemcpyAsync(w.Y.d(), w.X.d(), sizeof(double) * per * batch, cudaMemcpyDeviceToDevice, s));
        double* Y = w.Y.d();
        double* Yp = w.Yp.d();
        double* Yn = w.Yn.d();
        {
            StageTimer tf(w.basis ? "sq.filter" : "ss.filter", s);
            // columns below the smallest locked prefix of the filtered slices
            // are final: filter only [cf, b)
            int64_t cf = b;
            for (int64_t sl = 0; sl < batch; ++sl)
                if (deg[sl] > 0) cf = std::min<int64_t>(cf, nlock[sl]);
            if (cf >= b) cf = 0;
            const int64_t bf = b - cf;
            int64_t lmax = 0;
            for (int64_t sl = 0; sl < batch; ++sl)
                if (deg[sl] > 0) lmax = std::max<int64_t>(lmax, nlock[sl]);
            for (int j = 0; j < dmax; ++j) {
                // only the slices still filtering at this degree (compacted batch)
                const int na = nact[j];
                const int* zm = w.zmap.as<int>() + (int64_t)j * batch;
                const double* cfj = w.coef.d() + 3 * (int64_t)j * batch;
                // INT8 filter: the Chebyshev step rides on the product's store
                // (Yn = a (G Y) + b Y + c Yp straight from TMEM; columns below cf
                // of Yn are never read: locked in every filtering slice, they are
                // restored from X after the filter)
                const bool fused = oz_filter && !near_floor && bf <= 64;
                if (na > 0) {
                    // Z = G Y, P = X^T Y, Z -= X diag(theta_L) P   (columns [cf, b))
                    if (oz_filter && !near_floor) {
                        const bool split = bf <= 64 && nlo[j] + nl3[j] > 0;
                        // only the digit planes this degree's products read
                        const int planes = !split || nhi[j] > 0 ? 6 : (nlo[j] > 0 ? 4 : 3);
                        Yd.split(Y + cf * r, r, per, r, bf, r, batch, s, zm, na, 0, 0, nullptr, 6, 0, 0, nullptr,
                                 planes);
                        const int* zlo = w.zmap.as<int>() + (int64_t)(dmax + j) * batch;
                        const int* zhi = w.zmap.as<int>() + (int64_t)(2 * dmax + j) * batch;
                        const int* zl3 = w.zmap.as<int>() + (int64_t)(3 * dmax + j) * batch;
                        const ChebFuse cfu{Y + cf * r, Yp + cf * r, cfj};
                        const ChebFuse* cp = fused ? &cfu : nullptr;
                        double* out = fused ? Yn + cf * r : w.Z.d() + cf * r;
                        if (split) {
                            if (nl3[j] > 0) ozaki_gemm(Gd, Yd, nl3[j], zl3, out, r, per, s, 3, true, cp);
                            if (nlo[j] > 0) ozaki_gemm(Gd, Yd, nlo[j], zlo, out, r, per, s, 4, true, cp);
                            if (nhi[j] > 0) ozaki_gemm(Gd, Yd, nhi[j], zhi, out, r, per, s, 6, true, cp);
                        } else {
                            ozaki_gemm(Gd, Yd, na, zm, out, r, per, s, 6, true, cp);
                        }
                    } else {
                        gg(G, r, r * r, false, Y + cf * r, r, per, w.Z.d() + cf * r, r, per, r, bf, r, na, 1.0, 0.0,
                           s, zm, batch);
                    }
                    // deflation over the locked columns only (lmax: most locked among
                    // the filtered slices; none locked -> nothing to deflate)
                    if (lmax > 0) {
                        gg(w.X.d(), r, per, true, Y + cf * r, r, per, w.P.d(), lmax, lmax * bf, lmax, bf, r, na, 1.0,
                           0.0, s, zm, batch);
                        // fused: the correction lands on Yn, scaled by the slice's a
                        scale_rows_kernel<<<grid1(lmax * bf * batch), 256, 0, s>>>(
                            w.P.d(), w.wmask.d(), lmax, b, bf, lmax * bf * batch, fused ? cfj : nullptr);
                        count_launch();
                        gg(w.X.d(), r, per, false, w.P.d(), lmax, lmax * bf, (fused ? Yn : w.Z.d()) + cf * r, r, per,
                           r, bf, lmax, na, -1.0, 1.0, s, zm, batch);
                    }
                }
                // only the slices still filtering at this degree; a slice that
                // stops keeps its block in its own buffer of the rotation
                if (na > 0 && !fused) {
                    cheb_kernel<<<grid1(per * na), 256, 0, s>>>(Yn, w.Z.d(), Y, Yp, w.coef.d() + 3 * j * batch,
                                                                per, per * na, r, cf, zm);
                    count_launch();
                    check_launch("cheb");
                }
                double* t = Yp;  // rotate (Yp, Y, Yn) <- (Y, Yn, Yp)
                Yp = Y;
                Y = Yn;
                Yn = t;
            }
        }
        // slices that stopped early: their filtered block into the final buffer
        // (after d degrees a slice's block sits in rotation slot d % 3)
        {
            std::vector<int> gl;
            for (int64_t sl = 0; sl < batch; ++sl)
                if (deg[sl] > 0 && deg[sl] % 3 != dmax % 3) {
                    gl.push_back((int)sl);
                    gl.push_back(deg[sl] % 3);
                }
            if (!gl.empty()) {
                if ((int64_t)gl.size() * 4 > (int64_t)w.glist.bytes()) w.glist = DeviceBuffer(gl.size() * sizeof(int));
                PPC_CUDA_CHECK(cudaMemcpyAsync(w.glist.d(), gl.data(), sizeof(int) * gl.size(), cudaMemcpyHostToDevice, s));
                double* cyc[3] = {w.Y.d(), w.Yn.d(), w.Yp.d()};
                gather_filtered_kernel<<<dim3(64, (unsigned)(gl.size() / 2)), 256, 0, s>>>(
                    cyc[dmax % 3], cyc[0], cyc[1], cyc[2], w.glist.as<int>(), per);
                count_launch();
                check_launch("gather_filtered");
            }
        }
        // the slices still iterating (degree-0 list of the filter): the rest
        // are final and skip the orthonormalization and Rayleigh-Ritz
        const int nact0 = nact[0];
        const int* zact = w.zmap.as<int>();
        // locked columns back, normalize, CholQR2, Rayleigh-Ritz
        dim3 grid((unsigned)((b + 7) / 8), (unsigned)nact0);
        restore_normalize_kernel<<<grid, 256, 0, s>>>(Y, w.X.d(), w.nlock.as<int>(), r, b, zact);
        count_launch();
        check_launch("restore_normalize");
        // CholQR3 writes through w.Yn; make sure Y is not aliased with it
        if (Y == w.Yn.d()) {
            PPC_CUDA_CHECK(cudaMemcpyAsync(w.Yp.d(), Y, sizeof(double) * per * batch, cudaMemcpyDeviceToDevice, s));
            Y = w.Yp.d();
        }
        double* Xn = (Y == w.Y.d()) ? w.Yp.d() : w.Y.d();
        // Rayleigh-Ritz only on the columns past the common locked prefix
        int64_t c0 = b - 1;
        for (int64_t sl = 0; sl < batch; ++sl)
            if (deg[sl] > 0) c0 = std::min<int64_t>(c0, nlock[sl]);
        if (c0 > 0)  // locked columns of the basis are final: copy them through
            PPC_CUDA_CHECK(cudaMemcpy2DAsync(Xn, sizeof(double) * per, w.X.d(), sizeof(double) * per,
                                             sizeof(double) * r * c0, batch, cudaMemcpyDeviceToDevice, s));
        cholqr3(w, Y, Xn, c0, s, zact, nact0);
        // approximate Ritz pairs until something has converged (locking uses
        // true residuals, so an inexact early Rayleigh-Ritz cannot lock early)
        const bool early = it < 2 && c0 == 0;
        rayleigh_ritz(w, G, r * r, Xn, c0, s, gtol_rel, early ? 4 : 0, zact, nact0,
                      (oz_filter && !near_floor) ? &Gd : nullptr, &Yd);
    }
    // outputs: leading k Ritz pairs
    PPC_CUDA_CHECK(cudaMemcpy2DAsync(Xout, sizeof(double) * r * k, w.X.d(), sizeof(double) * per,
                                     sizeof(double) * r * k, batch, cudaMemcpyDeviceToDevice, s));
    PPC_CUDA_CHECK(cudaMemcpy2DAsync(lambda, sizeof(double) * k, w.th.d(), sizeof(double) * b,
                                     sizeof(double) * k, batch, cudaMemcpyDeviceToDevice, s));
}

bool subspace_svd(const double* A, int64_t m, int64_t n, int64_t stride, int64_t batch, int64_t k,
                  double* U, double* S, double* V, double* tail2, cudaStream_t s, const char* finite_who) {
    bool checked = false;
    const bool tall = m >= n;
    const int64_t r = tall ? n : m;  // Gram dimension
    DeviceBuffer G(sizeof(double) * r * r * batch);
    {
        StageTimer tg("ss.gram", s, (double)batch * r * r * (tall ? m : n), 8.0 * batch * m * n);
        // tall slices: G_b = A_b^T A_b is the Gram of an m-row tube matrix
        // (INT8 tensor-core Ozaki SYRK where eligible)
        // the split of the INT8 slice Grams reads every entry once: the
        // input's finiteness check (matrix_kernels.cpp:32) rides on it
        std::unique_ptr<FiniteFlag> ff;
        if (finite_who && tall) ff.reset(new FiniteFlag(s));
        const bool oz = tall && ozaki_syrk_batched(A, m, stride, m, n, batch, G.d(), s, ff ? ff->d() : nullptr);
        if (oz && ff) {
            ff->check(s, finite_who);
            checked = true;
        }
        if (!oz) {
            GemmDesc d;
            d.M = r; d.N = r; d.batch = batch; d.symmetric = true;
            d.C = G.d(); d.ldc = r; d.strideC = r * r;
            d.A = A; d.B = A; d.strideA = stride; d.strideB = stride;
            if (tall) {  // G = A^T A: A(mm,kk) = A[kk + mm*m], B(kk,nn) = A[kk + nn*m]
                d.K = m; d.lda = m; d.a_kmajor = true; d.ldb = m; d.b_nmajor = false;
            } else {     // G = A A^T: A(mm,kk) = A[mm + kk*m], B(kk,nn) = A[nn + kk*m]
                d.K = n; d.lda = m; d.a_kmajor = false; d.ldb = m; d.b_nmajor = true;
            }
            gemm(d, s);
        }
    }
    DeviceBuffer Xk(sizeof(double) * r * k * batch), lam(sizeof(double) * k * batch);
    // slice Grams up to 1024: the batched direct solver (one cooperative
    // launch tridiagonalizes every Gram); larger ones: subspace iteration
    static const bool direct = !(std::getenv("PPC_SLICE_TRIDIAG") && std::atoi(std::getenv("PPC_SLICE_TRIDIAG")) == 0);
    if (direct && tridiag_eig_preferred(r, k, batch))
        tridiag_eig_top_batched(G.d(), r, r * r, batch, k, Xk.d(), lam.d(), s);
    else
        subspace_eig_top(G.d(), r, batch, k, Xk.d(), lam.d(), s, true);
    // polish: W = A Xk (tall: m x k) or A^T Xk (wide: n x k)
    StageTimer tp("ss.polish", s);
    const int64_t o = tall ? m : n;
    DeviceBuffer Wb(sizeof(double) * o * k * batch), Qw(sizeof(double) * o * k * batch),
        T1(sizeof(double) * o * k * batch), Sk(sizeof(double) * k * k * batch),
        R1(sizeof(double) * k * k * batch), R2(sizeof(double) * k * k * batch),
        Ri(sizeof(double) * k * k * batch), R(sizeof(double) * k * k * batch),
        Ur(sizeof(double) * k * k * batch), Vr(sizeof(double) * k * k * batch), weak(sizeof(int) * batch);
    PPC_CUDA_CHECK(cudaMemsetAsync(weak.d(), 0, sizeof(int) * batch, s));
    {
        GemmDesc d;
        d.M = o; d.N = k; d.K = r; d.batch = batch;
        d.A = A; d.strideA = stride;
        d.lda = m;
        d.a_kmajor = !tall;  // wide: A^T (n x m): A(mm,kk) = A[kk + mm*m]
        d.B = Xk.d(); d.ldb = r; d.strideB = r * k;
        d.C = Wb.d(); d.ldc = o; d.strideC = o * k;
        gemm(d, s);
    }
    // CholQR2 of W (cond(W) = sigma_1/sigma_k): W = Qw R, R = R2 R1
    const size_t ksm = (size_t)k * k * sizeof(double);
    if (ksm > 48 * 1024)
        PPC_CUDA_CHECK(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ksm));
    g_AtB(Wb.d(), Wb.d(), Sk.d(), o, k, k, batch, o * k, o * k, s);
    chol_inv_kernel<<<(unsigned)batch, k > 16 ? 1024 : 256, ksm, s>>>(Sk.d(), Ri.d(), k, 0, nullptr, R1.d(), nullptr,
                                                                         weak.as<int>());
    count_launch();
    check_launch("chol_inv");
    g_AB(Wb.d(), Ri.d(), T1.d(), o, k, k, batch, o * k, k * k, 1.0, nullptr, 0.0, s);
    g_AtB(T1.d(), T1.d(), Sk.d(), o, k, k, batch, o * k, o * k, s);
    chol_inv_kernel<<<(unsigned)batch, k > 16 ? 1024 : 256, ksm, s>>>(Sk.d(), Ri.d(), k, 0, nullptr, R2.d(), nullptr,
                                                                         weak.as<int>());
    count_launch();
    check_launch("chol_inv");
    g_AB(T1.d(), Ri.d(), Qw.d(), o, k, k, batch, o * k, k * k, 1.0, nullptr, 0.0, s);
    g_AB(R2.d(), R1.d(), R.d(), k, k, k, batch, k * k, k * k, 1.0, nullptr, 0.0, s);
    {  // slices with a weak pivot: Qw and R again by CGS2 (one CTA each; the rest return at once)
        DeviceBuffer rowm(sizeof(double) * o * batch);
        cgs2_fallback_kernel<<<(unsigned)batch, 512, 0, s>>>(Wb.d(), Qw.d(), R.d(), o, (int)k, weak.as<int>(),
                                                             rowm.d());
        count_launch();
        check_launch("cgs2_fallback");
    }
    // R = Ur diag(sigma) Vr^T (one-CTA Jacobi, high relative accuracy)
    jacobi_svd(R.d(), k, k, k * k, batch, k, Ur.d(), S, Vr.d(), nullptr, s);
    if (tall) {  // A ~ (Qw Ur) sigma (Xk Vr)^T
        g_AB(Qw.d(), Ur.d(), U, m, k, k, batch, m * k, k * k, 1.0, nullptr, 0.0, s);
        g_AB(Xk.d(), Vr.d(), V, n, k, k, batch, n * k, k * k, 1.0, nullptr, 0.0, s);
    } else {     // A^T ~ (Qw Ur) sigma (Xk Vr)^T  =>  A ~ (Xk Vr) sigma (Qw Ur)^T
        g_AB(Xk.d(), Vr.d(), U, m, k, k, batch, m * k, k * k, 1.0, nullptr, 0.0, s);
        g_AB(Qw.d(), Ur.d(), V, n, k, k, batch, n * k, k * k, 1.0, nullptr, 0.0, s);
    }
    sign_rule(U, m, k, batch, V, n, s);  // matrix_kernels.cpp:16-25
    if (tail2) slice_tail_energy(A, m, n, stride, batch, k, U, S, V, tail2, s);
    return checked;
}

}  // namespace ppc
