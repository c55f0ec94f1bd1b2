// FP64 Gram on the INT8 tensor cores (Ozaki scheme, ozaki.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

#include "internal.h"

namespace ppc {

// Ozaki digits of nblk FP64 blocks of at most KC <= 4096 rows: block c is
// X + c*stride (batched; its first min(KC, rows) rows), or, with stride 0,
// sub-block c % per of plan chunk c / per (chunk rows each) of one matrix
// (leading dimension ldx). Every column of a block is scaled by a power of
// two and cut into 6 8-bit digits along the rows (the K dimension of the
// products below): a signed lead digit and five unsigned ones.
struct OzakiDigits {
    DeviceBuffer D, sc, sq;  // int8 planes [blk][digit][col][KCp]; scales, sums of squares [blk][col]
    int64_t rows = 0, cols = 0, KCp = 0, nblk = 0;
    int nd = 6;              // digit planes per block (6; 7 adds 8 bits for products with cancellation)
    bool uniform = false;    // block b holds rows [4096 b, 4096 b + 4096) of one matrix (row-chunked split)
    // zmap (device, nz entries; batched blocks only): split just those blocks
    void split(const double* X, int64_t ldx, int64_t stride, int64_t rows, int64_t cols, int64_t KC, int64_t nblk,
               cudaStream_t s, const int* zmap = nullptr, int64_t nz = 0, int64_t chunk = 0, int64_t per = 0,
               int* nonfinite = nullptr, int ndig = 6, int64_t block_base = 0, int64_t alloc_blocks = 0,
               const double* fixed_max = nullptr, int nwrite = 0, bool trans_src = false,
               const double* rowscale = nullptr);
    // fixed_max (device, per block): a bound on max|x| over the whole block,
    // giving every column the same scale (symmetric operands, sym_a below).
    // block_base / alloc_blocks: this call's nblk_ blocks land at block_base of an
    // allocation of max(nblk_, alloc_blocks) blocks (streamed row groups).
    // nwrite (0: all): only the leading nwrite digit planes are written, for
    // operands of reduced-level products (levels <= nwrite read no others).
    // rowscale (batched blocks only): every block reads the same source X
    // (no b * stride) with row k scaled by rowscale[b * rows + k].
    // trans_src (batched blocks only): element (k, c) of block b is
    // X[b * stride + c + k * ldx], the transpose of the usual layout.
};

// C_b (A.cols x B.cols, (m, n) at m + n*ldc, b at blk*strideC) = A_blk^T B_blk
// for the nbatch blocks blk = zmap[b] (or b): the FP64 product of the two
// split operands on the INT8 tensor cores (exact int32 digit-level sums).
// levels = 4 / 3 (B.cols <= 64 only) keep digit pairs of levels <= 5 / 4:
// ~1e-9 / ~1e-7 relative precision at 1/2 / 3/10 of the MMAs, for products
// that only steer an iteration (the Chebyshev filter far from convergence).
// sym_a: A's blocks are symmetric and split with one scale per block
// (fixed_max): A is streamed from its upper triangles only (half the reads).
// cheb (nullable, sym_a only): C = a (A^T B) + b Y + c Yp instead of A^T B,
// with Y and Yp laid out as C and the block's {a, b, c} at coef + 3 zmap[b]
// (one Chebyshev filter step fused into the store).
struct ChebFuse {
    const double* Y;
    const double* Yp;
    const double* coef;
};
void ozaki_gemm(const OzakiDigits& A, const OzakiDigits& B, int64_t nbatch, const int* zmap, double* C, int64_t ldc,
                int64_t strideC, cudaStream_t s, int levels = 6, bool sym_a = false, const ChebFuse* cheb = nullptr);
// Whether the Gram partials of a plan with chunks of `chunk` rows run on the
// integer path (a function of the plan only, see ozaki_gram_partials).
bool ozaki_gram_eligible(int64_t n3, int64_t chunk);
// The cheap dynamic-range gate of the INT8 products. The split rounds every
// value at ~2^-47 of its column's maximum, so an output C(a,b) carries an
// error ~ sqrt(K) 2^-46 max|A(a,:)| max|B(:,b)|, against FP64's ~ sqrt(K)
// 2^-53 |A(a,:)| |B(:,b)|: the two stay within a small factor while every
// row/column's peak ratio max|x| sqrt(K) / ||x|| is small (~3-4 for Gaussian
// data, sqrt(K) for a row dominated by one entry). Returns, per group of
// `group` consecutive columns of d, an upper bound (< 2x) on the largest
// peak ratio over all its blocks (one host sync).
std::vector<double> ozaki_peak_ratios(const OzakiDigits& d, int64_t K, int64_t group, cudaStream_t s);
// the same into device memory (out: ozaki_peak_groups(d, group) doubles), no sync
int64_t ozaki_peak_groups(const OzakiDigits& d, int64_t group);
void ozaki_peak_ratios_async(const OzakiDigits& d, int64_t K, int64_t group, double* out, cudaStream_t s);
constexpr double kOzakiPeakGate = 16.0;  // products whose operands exceed it run on FP64 DMMA
// The star product's inverse transform on the INT8 tensor cores: C (M x N,
// leading dimension ldc) = alpha A Q^T for A (M x K, leading dimension M) and
// Q (N x K), 32 <= K <= 64, N <= 256 a multiple of 32. A is split row-wise
// (one power-of-two scale per row over its K values: rows are independent,
// so row blocks and shards give the device call's bits); 21 digit pairs,
// error ~ sqrt(K) 2^-46 max|A(a,:)| max|Q(b,:)| <= 2^-43 |A(a,:)| |Q(b,:)|
// (row scaling bounds the peak ratio by sqrt(K)). false when not eligible
// (PPC_OZAKI_STAR_INV=0 disables).
bool ozaki_star_inverse_eligible(int64_t K, int64_t N);
bool ozaki_star_inverse(const double* A, int64_t M, int64_t K, const double* Q, int64_t N, double alpha, double* C,
                        int64_t ldc, cudaStream_t s);
// Whether the integer path applies to an output with M rows and K-length sums.
bool ozaki_gemm_eligible(int64_t M, int64_t K);
// the INT8 path is on (PPC_OZAKI / ppc_set_ozaki)
bool ozaki_path_on();

// {||X - Ch Q^T||^2, ||X||^2} for X (N x n3, leading dimension N), the
// reconstruction core Ch (N x p) and the basis Q (n3 x p): the core's digits
// per (4096-row block, slice) read MN-major, the scales folded into Q^T, a
// residual epilogue on the INT8 tensor cores. false when not eligible.
bool ozaki_recon_residual(const double* X, int64_t N, int64_t n3, const double* Ch, const double* Q, int64_t p,
                          double sums[2], cudaStream_t s);

// Per-plan-chunk partial Grams parts[c] = T_c^T T_c (nchunks x n3 x n3) of a
// tube matrix T (rows x n3, leading dimension ldT), as gram_partials, through
// 8-bit digit splitting and tcgen05 kind::i8 MMAs. Returns false when the
// shape is not eligible (caller falls back to the DMMA SYRK). PPC_OZAKI=0
// disables it. nonfinite (nullable device int): set to 1 if any value of T
// is NaN or Inf (the split reads every value once).
// keep (nullable): when the plan chunks are whole 4096-row blocks, T is split
// into 7 digits (the SYRK still uses 6 levels) and the digits are left in
// *keep for ozaki_mode3_forward.
// block_base / total_blocks: T is one row group of a larger matrix whose digits
// go to blocks [block_base, ...) of a total_blocks allocation in *keep (the
// caller sets keep->uniform once every group has landed).
bool ozaki_gram_partials(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk, int64_t nchunks,
                         double* parts, cudaStream_t s, int* nonfinite = nullptr, OzakiDigits* keep = nullptr,
                         int64_t block_base = 0, int64_t total_blocks = 0);

// out (N x p, leading dimension N) = T Q, the forward mode-3 transform, from
// T's retained 7-digit Gram digits td (read MN-major: pixels contiguous per
// column) and Q (n3 x p) with the per-(block, column) scales folded in: 28
// digit pairs, ~2^-55 of the per-block column scale, as accurate as FP64
// DMMA on the noise slices (where Ahat is ~1e-4 of |T||Q|). false when td
// does not qualify.
bool ozaki_mode3_forward(const OzakiDigits& td, int64_t N, const double* Q, int64_t p, double* out, cudaStream_t s);

// G_b (n x n, column-major, b < batch, stride n*n) = A_b^T A_b for A_b
// (rows x n, leading dimension lda) at A + b*strideA: the batched slice
// Grams. rows <= 4096. Returns false when not eligible.
// nonfinite (nullable device int): set to 1 if any entry of the rows x n
// blocks is NaN or Inf (the split reads every value once).
bool ozaki_syrk_batched(const double* A, int64_t lda, int64_t strideA, int64_t rows, int64_t n, int64_t batch,
                        double* G, cudaStream_t s, int* nonfinite = nullptr);

}  // namespace ppc
