// Small-panel kernels of the batched subspace iteration (subspace.cu): the
// r x bc (bc <= 64) panels of every slice, their bc x bc Grams, Cholesky
// factors and the panel-times-small-matrix products of CholQR and
// Rayleigh-Ritz.
//
// These products are short and many (78..128 slices, r = 2048, bc <= 64):
// the general DMMA GEMM ran them one 128 x 64 tile per slice (20 SMs idle,
// half of every tile padding) and the one-CTA Cholesky took 80-100 us on
// 64 x 64. Here:
//   panel_gram:  A^T B (upper triangle, mirrored) over split-K chunks of 128
//                rows, one CTA each, DMMA from shared memory; the partials
//                are summed in split order by a reduction kernel
//                (deterministic);
//   chol_inv64:  (shifted) Cholesky S = R^T R and R^{-1} for bc <= 64, one
//                256-thread CTA per slice, one barrier per step;
//   panel_apply: Y_out = Y_in * M (bc x bc) per slice, 64-row blocks, DMMA
//                with the A fragments loaded straight from HBM.
#include <algorithm>
#include <cmath>

#include "internal.h"
#include "panel.cuh"

namespace ppc {

namespace {

constexpr int kKc = 128;   // rows per split-K chunk / apply block
constexpr int kBc = 64;    // panel width bound

// Stage an nc x kn column block (column c of src at src + c*ld, kn <= kk
// rows used, zero padded to kk) into dst[c * dp + k], 16 loads of a thread in
// flight (a load-store loop leaves one DRAM round trip per element).
__device__ __forceinline__ void stage_cols(double* __restrict__ dst, int dp, const double* __restrict__ src,
                                           int64_t ld, int nc_valid, int nc, int kn, int kk) {
    const int n = nc * kk, nt = blockDim.x;
    for (int e0 = threadIdx.x; e0 < n; e0 += 16 * nt) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = e0 + u * nt;
            const int c = e / kk, k = e - c * kk;
            v[u] = (e < n && c < nc_valid && k < kn) ? __ldcs(src + (int64_t)c * ld + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = e0 + u * nt;
            const int c = e / kk, k = e - c * kk;
            if (e < n) dst[c * dp + k] = v[u];
        }
    }
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// Partial t (bc x bc, upper 16 x 16 tiles, at part + (t * zext + s) * bc^2)
// of A_s^T B_s over rows [128 t, 128 t + 128), slice s = zmap[blockIdx.y]
// (or blockIdx.y); panel_reduce_kernel sums the partials in split order.
// (A thread-block cluster of the nsplit CTAs reducing over DSMEM measured
// 145 us against 58: clusters of 16 co-schedule poorly.)
// Per CTA: one warp per 16 x 16 upper tile (2 x 2 DMMA m8n8k4 per 4-row k
// step); the chunk sits column-major in shared memory with a column stride
// of 132 doubles (= 4 mod 16), so every fragment read (lane g = column
// offset, t = k offset) hits each 8-byte bank pair exactly twice. A == B
// stages once.
constexpr int kGP = kKc + 4;
__global__ void __launch_bounds__(320) panel_gram_kernel(const double* __restrict__ A, int64_t sA,
                                                         const double* __restrict__ B, int64_t sB, int64_t r, int bc,
                                                         double* __restrict__ part, int64_t zext,
                                                         const int* __restrict__ zmap) {
    extern __shared__ double sm[];
    const int64_t s = zmap ? (int64_t)zmap[blockIdx.y] : (int64_t)blockIdx.y;
    const int t = blockIdx.x;
    const int64_t k0 = (int64_t)t * kKc;
    const int kn = (int)std::min<int64_t>(kKc, r - k0);
    const bool same = (A == B) && (sA == sB);
    double* As = sm;
    double* Bs = same ? sm : sm + kBc * kGP;
    const double* a = A + s * sA + k0;
    const double* b = B + s * sB + k0;
    const int ncol = (bc + 15) / 16 * 16;
    stage_cols(As, kGP, a, r, bc, ncol, kn, kKc);
    if (!same) stage_cols(Bs, kGP, b, r, bc, ncol, kn, kKc);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int nt = ncol / 16;
    // warp -> upper tile (ti, tj), column order
    int ti = warp, tj = 0;
    while (tj < nt && ti > tj) {
        ti -= tj + 1;
        ++tj;
    }
    double acc[2][2][2] = {};
    const bool live = tj < nt;
    const int i0 = 16 * ti, j0 = 16 * tj;
    if (live) {
        for (int kk = 0; kk < kKc; kk += 4) {
            double af[2], bf[2];
#pragma unroll
            for (int x = 0; x < 2; ++x) af[x] = As[(i0 + 8 * x + g) * kGP + kk + q];
#pragma unroll
            for (int y = 0; y < 2; ++y) bf[y] = Bs[(j0 + 8 * y + g) * kGP + kk + q];
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y) dmma884(acc[x][y], af[x], bf[y]);
        }
    }
    if (live) {
        double* o = part + ((int64_t)t * zext + s) * bc * bc;
        // C fragment: lane (g, q) holds (row g, columns 2q, 2q + 1) of each 8 x 8
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int i = i0 + 8 * x + g, j = j0 + 8 * y + 2 * q + h;
                    if (i < bc && j < bc) o[i + (int64_t)j * bc] = acc[x][y][h];
                }
    }
}

// S_s (full symmetric) = split-order sum of the nsplit partials' upper
// triangles, mirrored. CTA (c, z): entries e = c * 256 + thread of slice
// zmap[z]; all 16 loads of an entry in flight.
__global__ void __launch_bounds__(256) panel_reduce_kernel(const double* __restrict__ part, int nsplit, int64_t zext,
                                                           int bc, double* __restrict__ S,
                                                           const int* __restrict__ zmap) {
    const int64_t s = zmap ? (int64_t)zmap[blockIdx.y] : (int64_t)blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= bc * bc) return;
    const int i = e % bc, j = e / bc;
    if (i > j) return;
    const int64_t st = zext * bc * bc;
    const double* p = part + s * bc * bc + e;
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = u < nsplit ? p[u * st] : 0.0;
    double sum = v[0];
#pragma unroll
    for (int u = 1; u < 16; ++u)
        if (u < nsplit) sum += v[u];
    double* o = S + s * (int64_t)bc * bc;
    o[e] = sum;
    o[j + (int64_t)i * bc] = sum;
}

// One CTA (256 threads) per slice: S (bc x bc symmetric at S + s*bc*bc,
// the lower triangle read), optional shift 1e-15 trace(S); Cholesky
// S = R^T R (R upper) and R^{-1} (bc x bc, zeros below the diagonal) into
// Rinv. Right-looking, one barrier per step, the Cholesky of step k and the
// inverse's step k - 1 in the same pass:
//   W (working, lower)  : S, trailing updates W(i, j) -= W(i, k) W(j, k) / d_k
//   L (final, lower)    : column k = W(:, k) / sqrt(d_k), L(k, k) = sqrt(d_k)
//   B (lower)           : I, then B(i, j) -= L(i, k) X(k, j) (i > k >= j)
//   X = L^{-1} (lower)  : row k = B(k, :) / L(k, k)
// (each array is read and written in disjoint places within a step).
// Non-positive pivots use d = 1 (the unit pivot, as chol_inv_kernel), set
// fail; weak (nullable) flags pivots below 1e-12 of the largest diagonal.
__global__ void __launch_bounds__(256) chol_inv64_kernel(const double* __restrict__ S, int bc, int shift_pass,
                                                         double* __restrict__ Rinv, int* fail,
                                                         const int* __restrict__ zmap, int* __restrict__ weak) {
    constexpr int LD = kBc + 1;
    extern __shared__ double shm[];
    double* W = shm;
    double* L = W + kBc * LD;
    double* Bm = L + kBc * LD;
    double* X = Bm + kBc * LD;
    __shared__ double dv[kBc];  // 1 / L(k, k)
    __shared__ int bad;
    const int64_t s = zmap ? (int64_t)zmap[blockIdx.x] : (int64_t)blockIdx.x;
    const int tid = threadIdx.x;
    const double* S0 = S + s * (int64_t)bc * bc;
    for (int e = tid; e < bc * bc; e += blockDim.x) {
        const int i = e % bc, j = e / bc;
        if (i >= j) {
            W[i * LD + j] = S0[e];
            Bm[i * LD + j] = i == j ? 1.0 : 0.0;
        }
    }
    if (tid == 0) bad = 0;
    __syncthreads();
    double dmax = 0.0, sh = 0.0;
    {
        double tr = 0.0;
        for (int i = 0; i < bc; ++i) {  // every thread, same order
            tr += W[i * LD + i];
            dmax = fmax(dmax, W[i * LD + i]);
        }
        if (shift_pass) sh = 1e-15 * tr;
    }
    __syncthreads();
    if (shift_pass && tid < bc) W[tid * LD + tid] += sh;
    if (shift_pass) dmax += sh;
    __syncthreads();
    const int ti = tid & 15, tj = tid >> 4;
    for (int t = 0; t <= bc; ++t) {
        if (t < bc) {  // Cholesky step k = t
            const int k = t;
            const double d = W[k * LD + k];
            const bool ok = d > 0.0;
            const double dk = ok ? d : 1.0;
            const double rt = sqrt(dk), rs = 1.0 / rt, ri = 1.0 / dk;
            if (tid < bc && tid >= k) L[tid * LD + k] = tid == k ? rt : W[tid * LD + k] * rs;
            if (tid == 0) {
                dv[k] = rs;
                if (!ok) bad = 1;
                if (weak && !(d > 1e-12 * dmax)) weak[s] = 1;
            }
            // (i, j) = (k + 1 + ti + 16 a, k + 1 + tj + 16 b), j <= i: every
            // load of the step issued before the first store
            double wi[4], wjv[4], wv[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int i = k + 1 + ti + 16 * a, j = k + 1 + tj + 16 * a;
                wi[a] = i < bc ? W[i * LD + k] : 0.0;
                wjv[a] = j < bc ? W[j * LD + k] * ri : 0.0;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b2 = 0; b2 < 4; ++b2) {
                    const int i = k + 1 + ti + 16 * a, j = k + 1 + tj + 16 * b2;
                    wv[a][b2] = (i < bc && j <= i) ? W[i * LD + j] : 0.0;
                }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b2 = 0; b2 < 4; ++b2) {
                    const int i = k + 1 + ti + 16 * a, j = k + 1 + tj + 16 * b2;
                    if (i < bc && j <= i) W[i * LD + j] = fma(-wi[a], wjv[b2], wv[a][b2]);
                }
        }
        if (t >= 1) {  // inverse step k = t - 1 (L's column k and B's row k are final)
            const int k = t - 1;
            const double rk = dv[k];
            if (tid <= k) X[k * LD + tid] = Bm[k * LD + tid] * rk;
            double li[4], xk[4], bv[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int i = k + 1 + ti + 16 * a, j = tj + 16 * a;
                li[a] = i < bc ? L[i * LD + k] : 0.0;
                xk[a] = j <= k ? Bm[k * LD + j] * rk : 0.0;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b2 = 0; b2 < 4; ++b2) {
                    const int i = k + 1 + ti + 16 * a, j = tj + 16 * b2;
                    bv[a][b2] = (i < bc && j <= k) ? Bm[i * LD + j] : 0.0;
                }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b2 = 0; b2 < 4; ++b2) {
                    const int i = k + 1 + ti + 16 * a, j = tj + 16 * b2;
                    if (i < bc && j <= k) Bm[i * LD + j] = fma(-li[a], xk[b2], bv[a][b2]);
                }
        }
        __syncthreads();
    }
    // R^{-1} = X^T (upper)
    double* o = Rinv + s * (int64_t)bc * bc;
    for (int e = tid; e < bc * bc; e += blockDim.x) {
        const int i = e % bc, j = e / bc;
        o[e] = i <= j ? X[j * LD + i] : 0.0;
    }
    if (tid == 0 && bad && fail) atomicExch(fail, 1);
}

// Y_out rows [blockIdx.x * 64, +64) of slice s = Y_in rows * M_s (bc x bc
// at M + s*bc*bc, column-major). Y_in and Y_out are r x bc panels (leading
// dimension r) at per-slice strides sIn / sOut; they must not overlap.
// DMMA: warp w computes rows [8 w, 8 w + 8) x all bc columns (nb8 m8n8
// tiles). Each lane loads its A fragments for every k step straight from
// global memory before the first MMA (16 loads in flight: the kernel is
// load-latency bound; two CTAs per SM); M sits column-major in shared memory
// with a stride of 68 doubles (= 4 mod 16): conflict-free fragment reads.
constexpr int kAr = 64;  // rows per apply CTA
constexpr int kMP = kBc + 4;
__global__ void __launch_bounds__(256, 2) panel_apply_kernel(const double* __restrict__ Yin, int64_t sIn,
                                                             const double* __restrict__ M, double* __restrict__ Yout,
                                                             int64_t sOut, int64_t r, int bc,
                                                             const int* __restrict__ zmap) {
    __shared__ double Ms[kBc * kMP];  // Ms[c * kMP + l] = M(l, c)
    const int64_t s = zmap ? (int64_t)zmap[blockIdx.y] : (int64_t)blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * kAr;
    const int rn = (int)std::min<int64_t>(kAr, r - r0);
    const double* yi = Yin + s * sIn + r0;
    const double* ms = M + s * (int64_t)bc * bc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int m0 = 8 * warp;
    const int kpad = (bc + 3) / 4 * 4, nk = kpad / 4;
    double af[16];
    {
        const int row = m0 + g;
#pragma unroll
        for (int kb = 0; kb < 16; ++kb) {
            const int col = 4 * kb + q;
            af[kb] = (kb < nk && row < rn && col < bc) ? __ldcs(yi + (int64_t)col * r + row) : 0.0;
        }
    }
    const int npad = (bc + 7) / 8 * 8;
    stage_cols(Ms, kMP, ms, bc, bc, npad, bc, kpad);
    __syncthreads();
    const int nb8 = npad / 8;
    double acc[8][2] = {};
#pragma unroll
    for (int kb = 0; kb < 16; ++kb) {
        if (kb < nk) {
#pragma unroll
            for (int y = 0; y < 8; ++y)
                if (y < nb8) dmma884(acc[y], af[kb], Ms[(8 * y + g) * kMP + 4 * kb + q]);
        }
    }
    double* yo = Yout + s * sOut + r0;
#pragma unroll
    for (int y = 0; y < 8; ++y)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = m0 + g, c = 8 * y + 2 * q + h;
            if (y < nb8 && i < rn && c < bc) yo[(int64_t)c * r + i] = acc[y][h];
        }
}

}  // namespace

int panel_splits(int64_t r) { return (int)((r + kKc - 1) / kKc); }

// up to 16 split-K chunks of 128 rows (the consumers sum them in registers)
bool panel_kernels_ok(int64_t r, int64_t bc) { return bc >= 1 && bc <= kBc && r >= kKc && r <= 16 * kKc; }

void panel_gram(const double* A, int64_t sA, const double* B, int64_t sB, int64_t r, int64_t bc, int64_t batch,
                double* S, double* part, int64_t zext, const int* zmap, cudaStream_t s) {
    HostProf hp_("panel_gram");
    if (!panel_kernels_ok(r, bc)) fail(PPC_ARGUMENT, "panel_gram: shape");
    if (batch <= 0) return;
    const bool same = (A == B) && (sA == sB);
    const size_t smem = sizeof(double) * kBc * kGP * (same ? 1 : 2);
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, [] {
        PPC_CUDA_CHECK(cudaFuncSetAttribute(panel_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)(sizeof(double) * kBc * kGP * 2)));
    });
    const int nt = (int)((bc + 15) / 16);
    const int ns = panel_splits(r);
    const int64_t zx = std::max<int64_t>(zext, batch);
    panel_gram_kernel<<<dim3((unsigned)ns, (unsigned)batch), 32 * (nt * (nt + 1) / 2), smem, s>>>(
        A, sA, B, sB, r, (int)bc, part, zx, zmap);
    count_launch();
    check_launch("panel_gram");
    panel_reduce_kernel<<<dim3((unsigned)((bc * bc + 255) / 256), (unsigned)batch), 256, 0, s>>>(part, ns, zx,
                                                                                                (int)bc, S, zmap);
    count_launch();
    check_launch("panel_reduce");
}

void chol_inv64(const double* S, int64_t bc, int64_t batch, bool shift, double* Rinv, int* failed, const int* zmap,
                int* weak, cudaStream_t s) {
    HostProf hp_("chol_inv64");
    if (bc < 1 || bc > kBc) fail(PPC_ARGUMENT, "chol_inv64: bc out of range");
    if (batch <= 0) return;
    const size_t smem = sizeof(double) * 4 * kBc * (kBc + 1);
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, [&] {
        PPC_CUDA_CHECK(
            cudaFuncSetAttribute(chol_inv64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    chol_inv64_kernel<<<(unsigned)batch, 256, smem, s>>>(S, (int)bc, shift ? 1 : 0, Rinv, failed, zmap, weak);
    count_launch();
    check_launch("chol_inv64");
}

void panel_apply(const double* Yin, int64_t sIn, const double* M, double* Yout, int64_t sOut, int64_t r, int64_t bc,
                 int64_t batch, const int* zmap, cudaStream_t s) {
    HostProf hp_("panel_apply");
    if (!panel_kernels_ok(r, bc)) fail(PPC_ARGUMENT, "panel_apply: shape");
    if (batch <= 0) return;
    dim3 grid((unsigned)((r + kAr - 1) / kAr), (unsigned)batch);
    panel_apply_kernel<<<grid, 256, 0, s>>>(Yin, sIn, M, Yout, sOut, r, (int)bc, zmap);
    count_launch();
    check_launch("panel_apply");
}

}  // namespace ppc
