// FP64 tensor-core GEMM for sm_100a.
//
// Blackwell's tcgen05 has no f64 kind, so FP64 tensor-core math on B200 is
// the warp-level `mma.sync.aligned.m8n8k4.row.col.f64` (SASS DMMA.8x8x4),
// measured at 36.9 TFLOP/s chip-wide (MEASURED_FP64.json). This kernel:
//   - stages A/B tiles global->shared with cp.async (16 B when the operand is
//     2-aligned, 8 B otherwise) through a STAGES-deep ring;
//   - stores every tile in a "32-byte interleaved" layout: the operand's
//     contiguous dimension is cut into quads of 4 doubles, and each quad is
//     laid out contiguously along the other dimension:
//         idx(c, o) = ((c >> 2) * TO + o) * 4 + (c & 3)
//     so (a) a warp's cp.async writes 512 contiguous bytes and reads 32 B
//     sectors from global, and (b) every DMMA fragment read (lane g = row,
//     t = k) touches 16 distinct 8-byte bank pairs per half-warp, for both
//     MN-major and K-major operands — no padding, no bank conflicts;
//   - accumulates in registers and runs one of three epilogues:
//       STORE  D = alpha*acc + beta*Cin
//       RESID  sum((X - alpha*acc)^2), sum(X^2) per CTA (fused residual norm,
//              the reconstruction is never written)
//     with optional symmetric (SYRK) tiling and deterministic split-K.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace ppc {

enum { EPI_STORE = 0, EPI_RESID = 1 };

struct GemmParams {
    int64_t M, N, K;
    const double* A; int64_t lda, strideA;  // per-batch stride (doubles)
    const double* B; int64_t ldb, strideB;
    double* C; int64_t ldc, strideC;        // output (STORE)
    const double* Cin; int64_t ldcin, strideCin;  // beta term source (nullable)
    double alpha, beta;
    int64_t kchunk;       // K range per split (blockIdx.y)
    int64_t strideCsplit; // output stride between splits (STORE partials)
    const double* X; int64_t ldx, strideX;  // RESID reference
    double* partial;      // RESID: 2 doubles per CTA, CTA linear id order
    int tri;              // 1: only tiles with n_tile >= m_tile (SYRK), mirror on store
    int nfast;            // raster: 1 = n tile fastest
    // k-blocked operands (kshift > 0): a K-major operand stored as consecutive
    // blocks of 2^kshift rows, element (k, o) at (k >> kshift) * kbstride +
    // o * ld + (k & mask). Keeps each pipeline stage inside one block (TLB).
    int kshift;
    int64_t kbstride;
    const int* zmap;      // nullable: batch index indirection (blockIdx.z -> batch)
};

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int VEC>
__device__ __forceinline__ void cp_async(double* smem_dst, const double* gsrc, bool valid) {
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    const int src_size = valid ? VEC * 8 : 0;
    if constexpr (VEC == 2) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gsrc),
                     "r"(src_size));
    } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(gsrc),
                     "r"(src_size));
    }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Load one operand tile into the interleaved layout. The tile has contiguous
// dimension of size TC (global stride 1) and other dimension TO (global
// stride ld). (c0, o0) is the tile origin; (cmax, omax) the valid extents.
template <int TC, int TO, int VEC, int NT>
__device__ __forceinline__ void load_tile(double* s, const double* g, int64_t ld, int64_t c0,
                                          int64_t o0, int64_t cmax, int64_t omax, int kshift = 0,
                                          int64_t kbstride = 0) {
    constexpr int PER_QUAD = 4 / VEC;
    constexpr int CHUNKS = TC * TO / VEC;
#pragma unroll
    for (int it = 0; it < (CHUNKS + NT - 1) / NT; ++it) {
        const int id = threadIdx.x + it * NT;
        if (CHUNKS % NT != 0 && id >= CHUNKS) break;
        const int r = id / PER_QUAD, v = id % PER_QUAD;
        const int q = r / TO, o = r % TO;
        const int64_t gc = c0 + q * 4 + v * VEC, go = o0 + o;
        const bool ok = (gc < cmax) && (go < omax);
        const int64_t off = kshift ? ((gc >> kshift) * kbstride + (gc & ((1LL << kshift) - 1)) + go * ld)
                                   : gc + go * ld;
        const double* src = ok ? g + off : g;
        cp_async<VEC>(s + id * VEC, src, ok);
    }
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool AK, bool BNM,
          int VEC, int EPI>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32)
    dmma_gemm_kernel(const GemmParams P) {
    constexpr int NT = WARPS_M * WARPS_N * 32;
    constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
    constexpr int TM = WM / 8, TN = WN / 8;
    static_assert(WM % 8 == 0 && WN % 8 == 0 && BK % 4 == 0, "tile");
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + STAGES * BM * BK;

    // ---- tile coordinates
    const int64_t mtiles = (P.M + BM - 1) / BM, ntiles = (P.N + BN - 1) / BN;
    int64_t mt, nt;
    if (P.tri) {  // upper-triangular enumeration (nt >= mt), row-major
        int64_t t = blockIdx.x;
        mt = 0;
        while (t >= ntiles - mt) { t -= ntiles - mt; ++mt; }
        nt = mt + t;
    } else if (P.nfast) {
        nt = blockIdx.x % ntiles;
        mt = blockIdx.x / ntiles;
    } else {
        mt = blockIdx.x % mtiles;
        nt = blockIdx.x / mtiles;
    }
    const int64_t split = blockIdx.y, bz = P.zmap ? (int64_t)P.zmap[blockIdx.z] : (int64_t)blockIdx.z;
    const int64_t kb = split * P.kchunk;
    const int64_t ke = min(P.K, kb + P.kchunk);
    const double* A = P.A + bz * P.strideA;
    const double* B = P.B + bz * P.strideB;
    const int64_t m0 = mt * BM, n0 = nt * BN;
    const int ktiles = (int)((ke - kb + BK - 1) / BK);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp % WARPS_M, wn = warp / WARPS_M;

    auto load_stage = [&](int stage, int64_t k0) {
        double* as = As + stage * BM * BK;
        double* bs = Bs + stage * BK * BN;
        if constexpr (!AK)  // A(m,k) at A[m + k*lda]: contiguous m
            load_tile<BM, BK, VEC, NT>(as, A, P.lda, m0, k0, P.M, ke);
        else                // A(m,k) at A[k + m*lda]: contiguous k
            load_tile<BK, BM, VEC, NT>(as, A, P.lda, k0, m0, ke, P.M, P.kshift, P.kbstride);
        if constexpr (!BNM)  // B(k,n) at B[k + n*ldb]: contiguous k
            load_tile<BK, BN, VEC, NT>(bs, B, P.ldb, k0, n0, ke, P.N, P.kshift, P.kbstride);
        else                 // B(k,n) at B[n + k*ldb]: contiguous n
            load_tile<BN, BK, VEC, NT>(bs, B, P.ldb, n0, k0, P.N, ke);
    };

    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < ktiles) load_stage(st, kb + (int64_t)st * BK);
        cp_async_commit();
    }

    for (int kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + STAGES - 1;
            if (nk < ktiles) load_stage(nk % STAGES, kb + (int64_t)nk * BK);
            cp_async_commit();
        }
        const double* as = As + (kt % STAGES) * BM * BK;
        const double* bs = Bs + (kt % STAGES) * BK * BN;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[TM], bf[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const int m = wm * WM + i * 8 + g, k = kk + t;
                af[i] = AK ? as[((k >> 2) * BM + m) * 4 + (k & 3)]
                           : as[((m >> 2) * BK + k) * 4 + (m & 3)];
            }
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int n = wn * WN + j * 8 + g, k = kk + t;
                bf[j] = BNM ? bs[((n >> 2) * BK + k) * 4 + (n & 3)]
                            : bs[((k >> 2) * BN + n) * 4 + (k & 3)];
            }
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) dmma884(acc[i][j], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();

    // ---- epilogue
    if constexpr (EPI == EPI_STORE) {
        double* C = P.C + bz * P.strideC + split * P.strideCsplit;
        const double* Cin = P.Cin ? P.Cin + bz * P.strideCin : nullptr;
        const bool diag = P.tri && (mt == nt);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int64_t m = m0 + wm * WM + i * 8 + g;
                    const int64_t n = n0 + wn * WN + j * 8 + 2 * t + e;
                    if (m < P.M && n < P.N) {
                        if (diag && m > n) continue;
                        double v = P.alpha * acc[i][j][e];
                        if (Cin && P.beta != 0.0) v += P.beta * Cin[m + n * P.ldcin];
                        C[m + n * P.ldc] = v;
                        if (P.tri && m != n) C[n + m * P.ldc] = v;
                    }
                }
    } else {  // EPI_RESID
        const double* X = P.X + bz * P.strideX;
        double sd = 0.0, sx = 0.0;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int64_t m = m0 + wm * WM + i * 8 + g;
                    const int64_t n = n0 + wn * WN + j * 8 + 2 * t + e;
                    if (m < P.M && n < P.N) {
                        const double x = X[m + n * P.ldx];
                        const double d = x - P.alpha * acc[i][j][e];
                        sd = fma(d, d, sd);
                        sx = fma(x, x, sx);
                    }
                }
        // fixed-order block reduction
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            sd += __shfl_xor_sync(0xffffffffu, sd, off);
            sx += __shfl_xor_sync(0xffffffffu, sx, off);
        }
        __syncthreads();  // smem reuse
        double* red = smem;
        if (lane == 0) {
            red[warp * 2] = sd;
            red[warp * 2 + 1] = sx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = 0.0, b = 0.0;
            for (int w = 0; w < NT / 32; ++w) {
                a += red[w * 2];
                b += red[w * 2 + 1];
            }
            const int64_t cta = blockIdx.x + (int64_t)gridDim.x * (blockIdx.y + (int64_t)gridDim.y * blockIdx.z);
            P.partial[cta * 2] = a;
            P.partial[cta * 2 + 1] = b;
        }
    }
}

// ---------------------------------------------------------------- host API
// op(A): a_kmajor=false -> A is M x K col-major (lda >= M);
//        a_kmajor=true  -> A is stored K x M col-major (lda >= K), i.e. A^T.
// op(B): b_nmajor=false -> B is K x N col-major (ldb >= K);
//        b_nmajor=true  -> B is stored N x K col-major (ldb >= N), i.e. B^T.
struct GemmDesc {
    int64_t M = 0, N = 0, K = 0, batch = 1;
    const double* A = nullptr; int64_t lda = 0, strideA = 0; bool a_kmajor = false;
    const double* B = nullptr; int64_t ldb = 0, strideB = 0; bool b_nmajor = false;
    double* C = nullptr; int64_t ldc = 0, strideC = 0;
    const double* Cin = nullptr; int64_t ldcin = 0, strideCin = 0;
    double alpha = 1.0, beta = 0.0;
    bool symmetric = false;  // C = A^T A-style SYRK: only upper tiles, mirrored
    // split-K: > 1 writes `splits` partial outputs at C + s*strideCsplit
    int64_t splits = 1, strideCsplit = 0;
    int64_t kchunk = 0;  // rows of K per split; 0 = ceil(K / splits) rounded to 16
    int kshift = 0;      // k-blocked K-major operands (see GemmParams)
    int64_t kbstride = 0;
    const int* zmap = nullptr;  // device array of `batch` batch indices (nullable)
    int64_t zmap_extent = 0;    // with zmap: number of batches the indices refer to
    bool allow_ws = true;       // may use the warp-specialized TMA kernel
};

// Warp-specialized persistent TMA kernel (gemm_ws.cu); false = not eligible.
bool gemm_ws(const GemmDesc& d, int epi, const double* X, int64_t ldx, int64_t strideX, double* partials,
             int64_t* ctas_out, cudaStream_t s);

// D = alpha op(A) op(B) + beta Cin (EPI_STORE).
void gemm(const GemmDesc& d, cudaStream_t s);
// Fused residual: per-CTA partial sums of (X - alpha op(A)op(B))^2 and X^2.
// Returns the number of CTAs (partials has room for 2*ctas doubles).
int64_t gemm_residual_ctas(const GemmDesc& d, const double* X, int64_t ldx, int64_t strideX);
void gemm_residual(const GemmDesc& d, const double* X, int64_t ldx, int64_t strideX,
                   double* partials, cudaStream_t s);

}  // namespace ppc
