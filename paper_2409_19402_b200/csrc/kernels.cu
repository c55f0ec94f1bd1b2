// Memory-bound helper kernels (see kernels.cuh).
#include "internal.h"
#include "kernels.cuh"

namespace ppc {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order two-value block reduction (blockDim.x multiple of 32, <= 1024).
__device__ __forceinline__ void block_sum2(double& a, double& b) {
    __shared__ double red[2][32];
    a = warp_sum(a);
    b = warp_sum(b);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        red[0][w] = a;
        red[1][w] = b;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        a = l < nw ? red[0][l] : 0.0;
        b = l < nw ? red[1][l] : 0.0;
        a = warp_sum(a);
        b = warp_sum(b);
    }
}

__global__ void __launch_bounds__(kReduceThreads)
    sumsq_partials_kernel(const double* __restrict__ a, const double* __restrict__ b,
                          int64_t count, double* __restrict__ partials) {
    double sd = 0.0, sa = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b) {
        for (; i + 3 * stride < count; i += 4 * stride) {
            double x0 = a[i], x1 = a[i + stride], x2 = a[i + 2 * stride], x3 = a[i + 3 * stride];
            double d0 = x0 - b[i], d1 = x1 - b[i + stride], d2 = x2 - b[i + 2 * stride],
                   d3 = x3 - b[i + 3 * stride];
            sd = fma(d0, d0, sd); sd = fma(d1, d1, sd); sd = fma(d2, d2, sd); sd = fma(d3, d3, sd);
            sa = fma(x0, x0, sa); sa = fma(x1, x1, sa); sa = fma(x2, x2, sa); sa = fma(x3, x3, sa);
        }
        for (; i < count; i += stride) {
            const double x = a[i], d = x - b[i];
            sd = fma(d, d, sd);
            sa = fma(x, x, sa);
        }
    } else {
        for (; i + 3 * stride < count; i += 4 * stride) {
            double x0 = a[i], x1 = a[i + stride], x2 = a[i + 2 * stride], x3 = a[i + 3 * stride];
            sa = fma(x0, x0, sa); sa = fma(x1, x1, sa); sa = fma(x2, x2, sa); sa = fma(x3, x3, sa);
        }
        for (; i < count; i += stride) sa = fma(a[i], a[i], sa);
        sd = sa;
    }
    block_sum2(sd, sa);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = sd;
        partials[2 * blockIdx.x + 1] = sa;
    }
}

__global__ void __launch_bounds__(1024) reduce_pairs_kernel(const double* __restrict__ p, int64_t n,
                                                           double* __restrict__ out) {
    double a = 0.0, b = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        a += p[2 * i];
        b += p[2 * i + 1];
    }
    block_sum2(a, b);
    if (threadIdx.x == 0) {
        out[0] = a;
        out[1] = b;
    }
}

__global__ void scale_columns_kernel(const double* __restrict__ U, const double* __restrict__ S,
                                     double* __restrict__ out, int64_t rows, int64_t k,
                                     int64_t total) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t col = i / rows;  // = j + b*k, the index into S (k x batch)
        out[i] = U[i] * S[col];
    }
}

__global__ void scale_columns_strided_kernel(const double* __restrict__ U, const double* __restrict__ S,
                                             double* __restrict__ out, int64_t rows, int64_t k, int64_t kmax,
                                             int64_t total) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t r = i % rows, jb = i / rows, j = jb % k, b = jb / k;
        out[i] = U[r + (j + b * kmax) * rows] * S[j + b * kmax];
    }
}

__global__ void truncate_columns_kernel(double* __restrict__ X, int64_t rows, int64_t r,
                                        const int64_t* __restrict__ rank, int64_t total) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t jb = i / rows, j = jb % r, b = jb / r;
        if (j >= rank[b]) X[i] = 0.0;
    }
}

__global__ void transpose_kernel(const double* __restrict__ in, double* __restrict__ out,
                                 int64_t rows, int64_t cols) {
    __shared__ double tile[32][33];
    const int64_t b = blockIdx.z;
    in += b * rows * cols;
    out += b * rows * cols;
    const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int64_t r = r0 + threadIdx.x, c = c0 + j;
        if (r < rows && c < cols) tile[j][threadIdx.x] = in[r + c * rows];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int64_t c = c0 + threadIdx.x, r = r0 + j;
        if (r < rows && c < cols) out[c + r * cols] = tile[threadIdx.x][j];
    }
}

__global__ void scale_kernel(double* x, int64_t n, double alpha) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) x[i] *= alpha;
}

__global__ void nonfinite_kernel(const double* __restrict__ x, int64_t n, int* flag) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        bad |= !isfinite(x[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(flag, 1);
}

unsigned grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    return (unsigned)g;
}

// Residual sums of a tall product with a short inner dimension:
// {sum (X - C B)^2, sum X^2} for C (M x K, column-major, lda), B(k, n) =
// Bq[n + k * ldb] and X (M x Nn, ldx), K <= KMAX. One thread per row: its K
// coefficients stay in registers, a CTA's column chunk of B sits in shared
// memory (read as broadcasts), and X streams through once, coalesced along
// the rows. HBM-bound (the residual GEMM's 128 x 128 tiles spend their time in
// a latency-exposed epilogue when K is 16-32: 0.3 ms at cfg2 against 0.03).
// Fixed grid and a fixed-order block sum: deterministic.
constexpr int kSkRows = 128;  // rows per CTA = threads
constexpr int kSkCols = 64;   // columns per CTA
// KP: K padded to a multiple of 4 with zero coefficients and zero B rows
// (fma(-0, 0, d) = d: the padding changes no bit), so the inner products are
// fully unrolled without predicates and B comes from shared memory two values
// per load (ncu on the first version: one LDS and one ISETP per DFMA, 45% of
// the stalls on the LDS results).
template <int KP>
__global__ void __launch_bounds__(kSkRows) smallk_residual_kernel(
    const double* __restrict__ Cm, int64_t lda, const double* __restrict__ Bq, int64_t ldb,
    const double* __restrict__ X, int64_t ldx, int64_t M, int64_t Nn, int K, double* __restrict__ partials) {
    __shared__ __align__(16) double bs[kSkCols * KP];  // bs[c * KP + k] = B(k, n0 + c), zero for k >= K
    const int64_t r = (int64_t)blockIdx.x * kSkRows + threadIdx.x;
    const int64_t n0 = (int64_t)blockIdx.y * kSkCols;
    const int nc = (int)(Nn - n0 < kSkCols ? Nn - n0 : kSkCols);
    for (int t = threadIdx.x; t < nc * KP; t += kSkRows) {
        const int c = t % nc, k = t / nc;  // consecutive threads: consecutive n (coalesced)
        bs[c * KP + k] = k < K ? Bq[n0 + c + (int64_t)k * ldb] : 0.0;
    }
    double cr[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) cr[k] = (k < K && r < M) ? Cm[r + (int64_t)k * lda] : 0.0;
    __syncthreads();
    double sd = 0.0, sa = 0.0;
    if (r < M) {
        const double* xp = X + r + n0 * ldx;
        constexpr int U = 8;
        int c = 0;
        for (; c + U <= nc; c += U) {
            double x[U], d[U];
#pragma unroll
            for (int u = 0; u < U; ++u) d[u] = x[u] = xp[(int64_t)(c + u) * ldx];
#pragma unroll
            for (int k = 0; k < KP; k += 2) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const double2 b2 = *reinterpret_cast<const double2*>(bs + (c + u) * KP + k);
                    d[u] = fma(-cr[k], b2.x, d[u]);
                    d[u] = fma(-cr[k + 1], b2.y, d[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                sd = fma(d[u], d[u], sd);
                sa = fma(x[u], x[u], sa);
            }
        }
        for (; c < nc; ++c) {
            const double xv = xp[(int64_t)c * ldx];
            double d = xv;
#pragma unroll
            for (int k = 0; k < KP; k += 2) {
                const double2 b2 = *reinterpret_cast<const double2*>(bs + c * KP + k);
                d = fma(-cr[k], b2.x, d);
                d = fma(-cr[k + 1], b2.y, d);
            }
            sd = fma(d, d, sd);
            sa = fma(xv, xv, sa);
        }
    }
    block_sum2(sd, sa);
    if (threadIdx.x == 0) {
        const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
        partials[2 * cta] = sd;
        partials[2 * cta + 1] = sa;
    }
}

}  // namespace

int64_t smallk_residual_ctas(int64_t M, int64_t Nn) {
    return ((M + kSkRows - 1) / kSkRows) * ((Nn + kSkCols - 1) / kSkCols);
}

void launch_smallk_residual(const double* Cm, int64_t lda, const double* Bq, int64_t ldb, const double* X,
                            int64_t ldx, int64_t M, int64_t Nn, int64_t K, double* partials, cudaStream_t s) {
    const dim3 grid((unsigned)((M + kSkRows - 1) / kSkRows), (unsigned)((Nn + kSkCols - 1) / kSkCols));
#define PPC_SMALLK(KP_)                                                                                            \
    smallk_residual_kernel<KP_><<<grid, kSkRows, 0, s>>>(Cm, lda, Bq, ldb, X, ldx, M, Nn, (int)K, partials)
    switch ((K + 3) / 4) {
        case 1: PPC_SMALLK(4); break;
        case 2: PPC_SMALLK(8); break;
        case 3: PPC_SMALLK(12); break;
        case 4: PPC_SMALLK(16); break;
        case 5: PPC_SMALLK(20); break;
        case 6: PPC_SMALLK(24); break;
        case 7: PPC_SMALLK(28); break;
        default: PPC_SMALLK(32); break;
    }
#undef PPC_SMALLK
    count_launch();
    check_launch("smallk_residual");
}

void launch_sumsq_partials(const double* a, const double* b, int64_t count, double* partials,
                           cudaStream_t s) {
    sumsq_partials_kernel<<<kReduceBlocks, kReduceThreads, 0, s>>>(a, b, count, partials);
    count_launch();
    check_launch("sumsq_partials");
}

void launch_reduce_pairs(const double* partials, int64_t n, double* out, cudaStream_t s) {
    reduce_pairs_kernel<<<1, 1024, 0, s>>>(partials, n, out);
    count_launch();
    check_launch("reduce_pairs");
}

void launch_scale_columns(const double* U, const double* S, double* out, int64_t rows,
                          int64_t k, int64_t batch, cudaStream_t s) {
    const int64_t total = rows * k * batch;
    if (!total) return;
    scale_columns_kernel<<<grid_for(total, 256), 256, 0, s>>>(U, S, out, rows, k, total);
    count_launch();
    check_launch("scale_columns");
}

void launch_scale_columns_strided(const double* U, const double* S, double* out, int64_t rows, int64_t k,
                                  int64_t kmax, int64_t batch, cudaStream_t s) {
    const int64_t total = rows * k * batch;
    if (!total) return;
    scale_columns_strided_kernel<<<grid_for(total, 256), 256, 0, s>>>(U, S, out, rows, k, kmax, total);
    count_launch();
    check_launch("scale_columns_strided");
}

void launch_truncate_columns(double* X, int64_t rows, int64_t r, int64_t batch, const int64_t* rank,
                             cudaStream_t s) {
    const int64_t total = rows * r * batch;
    if (!total) return;
    truncate_columns_kernel<<<grid_for(total, 256), 256, 0, s>>>(X, rows, r, rank, total);
    count_launch();
    check_launch("truncate_columns");
}

void launch_transpose(const double* in, double* out, int64_t rows, int64_t cols, int64_t batch,
                      cudaStream_t s) {
    if (!rows || !cols || !batch) return;
    dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32), (unsigned)batch);
    transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(in, out, rows, cols);
    count_launch();
    check_launch("transpose");
}

void launch_scale(double* x, int64_t n, double alpha, cudaStream_t s) {
    if (!n) return;
    scale_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, alpha);
    count_launch();
    check_launch("scale");
}

void launch_nonfinite(const double* x, int64_t n, int* flag, cudaStream_t s) {
    if (!n) return;
    nonfinite_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, flag);
    count_launch();
    check_launch("nonfinite");
}

}  // namespace ppc
