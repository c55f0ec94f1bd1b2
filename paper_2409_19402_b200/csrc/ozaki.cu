// FP64 products on the INT8 tensor cores (tcgen05 kind::i8): the Ozaki
// scheme (Ozaki, Ogita, Oishi, Rump 2012; the INT8 form of Ootomo, Ozaki and
// Yokota 2024), for the Grams and the Chebyshev filter products of the
// tSVDQ path.
//
// Split. Per block of at most KC = 4096 rows and per column j, the column is
// scaled by sigma_j = 2^e with max|x| / sigma_j < 1/2, rounded to nearest at
// 2^{-47} sigma_j and cut exactly into S = 6 balanced signed 8-bit digits:
//     x / sigma = 2^{-7} ( d_1 + 2^{-8} d_2 + ... + 2^{-40} d_6 ) + O(2^{-48}),
//     d_1 in [-64, 64], d_s in [-128, 127]
// (the unsigned base-256 digits of 128 x / sigma + c with c = 128 sum_s
// 2^{-8(s-1)}, each shifted by -128; every step is exact in FP64). Balanced
// digits keep the dropped low-order pair products sign-symmetric: with
// unsigned digits they are all positive and their chunk sums grew ~K,
// measured 8e-13 of max|G| instead of ~1e-14. The one exception is a Gram's
// diagonal, whose dropped same-digit products (d_4 d_4 at level 8, ...) are
// squares; it is taken from FP64 column sums of squares instead.
// Products. For C = A^T B over one block,
//     C(a,b) ~= sigma_a sigma_b sum_{L=2}^{S+1} 2^{-14-8(L-2)} Q_L(a,b),
//     Q_L = sum_{s+t=L} D_s^T D_t       (21 digit pairs, 6 levels),
// and every Q_L is an exact int32 sum (4096 * 6 * 128^2 < 2^31), accumulated
// by tcgen05.mma in its own TMEM accumulator. Between blocks the epilogue warps drain the levels
// (smallest weight first), apply the block's scales and add into FP64
// register accumulators, so one work item covers any number of blocks in a
// fixed order (deterministic, independent of sharding).
//
// Kernels: ozaki_split_kernel (one CTA per (block, column), block staged in
// shared memory: one HBM read), ozaki_mma_kernel (one TMA producer warp, one
// MMA-issuing warp, eight epilogue warps; TMA SWIZZLE_64B tiles of all six
// digit planes of A (128 rows) and B (80 rows) per 64-byte K stage, 20 MMAs
// of 128 x {80,160,240} x 32 per stage).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "internal.h"
#include "kernels.cuh"
#include "ozaki.h"
#include "umma_i8.cuh"

namespace ppc {

namespace {

using namespace umma;

constexpr int kS = 6;           // digits per value: signed lead + 5 balanced 8-bit
constexpr int kSmax = 7;        // digit planes of a 7-digit split (the Gram digits the transform reuses)
constexpr int kBM = 128;        // UMMA M
constexpr int kBN = 80;         // UMMA N: 6 level accumulators x 80 = 480 TMEM columns
constexpr int kBK = 64;         // bytes (= int8 elements) of K per stage, SWIZZLE_64B
constexpr int kStages = 2;       // (the 80-wide 6-level configuration)
// TMA ring depth per configuration: as many 64-byte K stages as fit ~221 KB
// of shared memory, 2..kMaxStages (80x6: 2, 64x7: 2, 64x6: 3, 64x4: 4, 64x3: 6)
constexpr int kMaxStages = 6;
constexpr int stages_for(int bn, int nl) {
    return (221 * 1024) / (nl * (kBM + bn) * kBK) < 2 ? 2
           : ((221 * 1024) / (nl * (kBM + bn) * kBK) > kMaxStages ? kMaxStages
                                                                 : (221 * 1024) / (nl * (kBM + bn) * kBK));
}
constexpr int64_t kKC = 4096;   // rows per exact int32 accumulation
constexpr int kEpiWarps = 8;    // two per TMEM lane quadrant, 40 columns each
constexpr int kThreads = (2 + kEpiWarps) * 32;
static_assert(kS * kBN <= 512, "TMEM budget");
static_assert(kBN / 2 == 40, "epilogue column split (32 + 8)");

// ------------------------------------------------------------------ split
// One CTA per (block b, column j). Row-chunked mode (stride == 0): block b is
// sub-block u = b % per of plan chunk cp = b / per, rows
// [cp*chunk + u*KC, min(cp*chunk + (u+1)*KC, (cp+1)*chunk, rows)). Batched
// mode: block b is the first min(KC, rows) rows of X + b*stride.
// D layout: [(b*S + s)*cols + j][KCp] bytes; scale[b*cols + j].
// CPB columns per CTA (CPB * KCp <= 4096): 256 / CPB threads per column, so
// short blocks (the facewise / filter operands, K = 512 .. 2048) still keep
// 16 loads per thread in flight.
// TRS: the source is transposed, element (k, c) of block b at
// X[b stride + c + k ldx] (the facewise product's A-hat slices, read in place
// of a transposed copy): loaded with the columns across the lanes (coalesced),
// staged, then reduced and split exactly as a column-major source.
template <int ND, int CPB, bool TRS = false>
__global__ void __launch_bounds__(256) ozaki_split_kernel(const double* __restrict__ X, int64_t ldx, int64_t stride,
                                                          int64_t rows, int64_t cols, int64_t KC, int64_t KCp,
                                                          int64_t chunk, int64_t per, int8_t* __restrict__ D,
                                                          double* __restrict__ scale, double* __restrict__ sumsq,
                                                          const int* __restrict__ zmap, int* __restrict__ nonfinite,
                                                          const double* __restrict__ fixed_max, int nwrite,
                                                          const double* __restrict__ rowscale) {
    // rowscale (nullable, batched blocks, not TRS): every block reads the SAME
    // source X and scales row k by rowscale[b * rows + k] (the forward
    // transform's diag(sigma_b) Q, without materializing it per block)
    constexpr int TPC = 256 / CPB;  // threads per column
    constexpr int WPC = TPC / 32;   // warps per column
    constexpr int SCOL = kKC / CPB + (TRS ? 1 : 0);  // staged column stride (+1: no bank conflicts)
    __shared__ double stage[TRS ? SCOL * CPB : kKC];
    const int cc = threadIdx.x / TPC, lt = threadIdx.x % TPC;
    const int64_t j = (int64_t)blockIdx.x * CPB + cc;
    const bool live = j < cols;
    const int64_t b = zmap ? zmap[blockIdx.y] : blockIdx.y;
    int64_t r0, len;
    if (stride) {
        r0 = 0;
        len = std::min<int64_t>(KC, rows);
    } else {
        const int64_t cp = b / per, u = b - cp * per;
        r0 = cp * chunk + u * KC;
        const int64_t end = std::min<int64_t>(std::min<int64_t>(r0 + KC, (cp + 1) * chunk), rows);
        len = std::max<int64_t>(0, end - r0);
    }
    if (!live) len = 0;
    double* stg = stage + cc * SCOL;
    // all 16 loads of a thread in flight before any use (the kernel is
    // DRAM-latency bound); same per-thread summation order as a strided loop
    double mx = 0.0, ss = 0.0;
    constexpr int NL = kKC / 256;
    double v[NL];
    if (TRS) {
        // lanes over the CPB columns, then over k; every column's full K
        // extent is staged before the per-column reductions read it back
        const int cl = threadIdx.x % CPB, kl = threadIdx.x / CPB;
        const int64_t jc = (int64_t)blockIdx.x * CPB + cl;
        const int64_t klen = jc < cols ? std::min<int64_t>(KC, rows) : 0;
        const double* src = X + b * stride + (jc < cols ? jc : 0);
#pragma unroll
        for (int q = 0; q < NL; ++q) {
            const int64_t i = kl + TPC * q;
            v[q] = i < klen ? __ldcs(src + i * ldx) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < NL; ++q)
            if (kl + TPC * q < kKC / CPB) stage[cl * SCOL + kl + TPC * q] = v[q];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NL; ++q) v[q] = stg[lt + TPC * q];
    } else {
        const double* col = X + (stride && !rowscale ? b * stride : 0) + (live ? j : 0) * ldx + r0;
#pragma unroll
        for (int q = 0; q < NL; ++q) {
            const int64_t i = lt + TPC * q;
            v[q] = i < len ? __ldcs(col + i) : 0.0;
        }
        if (rowscale) {
            const double* rs = rowscale + b * rows + r0;
#pragma unroll
            for (int q = 0; q < NL; ++q) {
                const int64_t i = lt + TPC * q;
                if (i < len) v[q] = rs[i] * v[q];
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NL; ++q) {
        if (!TRS) stg[lt + TPC * q] = v[q];
        mx = fmax(mx, fabs(v[q]));
        ss = fma(v[q], v[q], ss);
    }
    // column max and (fixed-order) sum of squares: the Gram diagonal in FP64
    __shared__ double red[8], red2[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5] = mx;
        red2[threadIdx.x >> 5] = ss;
    }
    __syncthreads();
    __shared__ double colmax[CPB];
    if (lt < 32) {
        mx = lt < WPC ? red[cc * WPC + lt] : 0.0;
        ss = lt < WPC ? red2[cc * WPC + lt] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            ss += __shfl_xor_sync(0xffffffffu, ss, o);
        }
        if (lt == 0) {
            colmax[cc] = mx;
            if (live) sumsq[b * cols + j] = ss;
            // the caller's finiteness check rides on this pass over the input:
            // an Inf makes the max Inf, a NaN makes the sum of squares NaN
            if (live && nonfinite && (!(mx <= 1.7976931348623157e308) || isnan(ss))) *nonfinite = 1;
        }
    }
    __syncthreads();
    if (!live) return;
    mx = fixed_max ? fixed_max[b] : colmax[cc];  // a block-wide bound: one scale for every column
    // sigma = 2^e > 2 max |x| (mx = 0: all digits zero)
    const int e = mx > 0.0 ? ilogb(mx) + 2 : 0;
    if (lt == 0) scale[b * cols + j] = mx > 0.0 ? ldexp(1.0, e) : 0.0;
    int8_t* out = D + ((b * ND) * cols + j) * KCp;
    const int64_t plane = cols * KCp;
    // Integer digit extraction with SH = 8 (ND - 1): y = rint(2^SH * 128 x / sigma)
    // (|y| < 2^(SH+6)), U = y + c 2^SH with c 2^SH = 0x80...80 (ND - 1 bytes);
    // the lead digit is U >> SH (arithmetic: floor) and the balanced low
    // digits are the bytes of U ^ 0x80...80 (u - 128 as int8).
    constexpr int SH = 8 * (ND - 1);
    constexpr unsigned long long C80 = 0x8080808080808080ULL >> (64 - SH);
    // 2^(SH+7-e) as two finite factors: e may be near -1074 (subnormal columns)
    const int e1 = (SH + 7 - e) / 2;
    const double scl1 = mx > 0.0 ? ldexp(1.0, e1) : 0.0, scl2 = ldexp(1.0, SH + 7 - e - e1);
    for (int64_t i4 = (int64_t)lt * 4; i4 < KCp; i4 += (int64_t)TPC * 4) {
        uint32_t w[ND];
#pragma unroll
        for (int s = 0; s < ND; ++s) w[s] = 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t i = i4 + q;
            const long long y = i < len ? __double2ll_rn(stg[i] * scl1 * scl2) : 0LL;
            const long long U = y + (long long)C80;
            const uint64_t low = (uint64_t)U ^ C80;
            w[0] |= (uint32_t)(uint8_t)(int8_t)(U >> SH) << (8 * q);
#pragma unroll
            for (int s = 1; s < ND; ++s) w[s] |= (uint32_t)((low >> (SH - 8 * s)) & 0xFFu) << (8 * q);
        }
#pragma unroll
        for (int s = 0; s < ND; ++s)
            if (s < nwrite) *reinterpret_cast<uint32_t*>(out + s * plane + i4) = w[s];
    }
}

// ---------------------------------------------------------------- products
// One launch covers nbatch * tiles work items: item -> batch bi, tile t;
// bi -> output block ob (zmap, else bi), whose digit blocks are
// ob*per .. ob*per + per - 1 in both operands (summed in that order).
// SYM: the tiles are the upper triangle of an M x M Gram (A = B), each
// written together with its mirror.
struct OzParams {
    int64_t M, N;          // output extents per block
    int64_t mtiles, tiles; // row tiles; tiles per output block
    int64_t KCp;           // padded rows per digit block (multiple of kBK)
    int64_t per;           // digit blocks per output block
    int64_t nd;            // digit planes per block of both operands (6, or 7 for 7-digit splits)
    const int* zmap;       // nullable batch -> output block map
    const double* sa;      // row scales [digit block][M]
    const double* sb;      // column scales [digit block][N]
    const double* sq;      // SYM: column sums of squares [digit block][M] (the diagonal)
    double* C;             // output block ob at C + ob*strideC, (m, n) at m + n*ldc
    int64_t ldc, strideC;
    // RESID: instead of C, per-CTA sums {(X - C)^2, X^2} into partial[2*cta]
    // with X block ob at X + ob*strideX, (m, n) at m + n*ldx, rows
    // ob*M + m < m_total
    const double* X;
    int64_t ldx, strideX, m_total;
    double* partial;
    // Chebyshev step fused into the store (SYMA products only; cy nullable):
    // C = a (A^T B) + b Y + c Yp with Y, Yp laid out as C and the output
    // block's coefficients {a, b, c} at ccoef + 3 ob (subspace.cu's filter)
    const double* cy = nullptr;
    const double* cyp = nullptr;
    const double* ccoef = nullptr;
};

// tile t (upper-triangle order) -> (mb, nb): column tile nb holds
// min(floor((nb*BN + BN - 1) / kBM) + 1, mtiles) row tiles.
template <int BN>
__device__ __forceinline__ void tri_tile(int64_t t, int64_t mtiles, int64_t& mb, int64_t& nb) {
    nb = 0;
    for (;;) {
        const int64_t cnt = std::min<int64_t>((nb * BN + BN - 1) / kBM + 1, mtiles);
        if (t < cnt) break;
        t -= cnt;
        ++nb;
    }
    mb = t;
}


// Work item -> (output block ob, row tile mb, column tile nb).
template <bool SYM, int BN = kBN>
__device__ __forceinline__ void decode_item(const OzParams& P, int64_t item, int64_t& ob, int64_t& mb, int64_t& nb) {
    const int64_t bi = item / P.tiles;
    ob = P.zmap ? P.zmap[bi] : bi;
    if (SYM) {
        tri_tile<BN>(item - bi * P.tiles, P.mtiles, mb, nb);
    } else {
        const int64_t t = item - bi * P.tiles;
        mb = t % P.mtiles;
        nb = t / P.mtiles;
    }
}

// Persistent: CTA c runs items c, c + gridDim.x, ... The producer's stage
// counter and the MMA / epilogue block counter run on across items, so the
// next item's operands stream in while the current one is drained; one TMEM
// allocation serves every item. AMN: the A digits are MN-major ([plane][k][m],
// m contiguous), loaded as two 64-byte x 64-row boxes per digit (LBO 4096 B).
// BN: output tile width (UMMA N per digit; 80, or 64 for 64-column panels);
// NL: digit levels computed (levels 2..NL+1, digits 1..NL of each operand:
// kS = full FP64 accuracy; fewer give ~2^(-8 NL + 1) relative precision for
// products that only steer an iteration).
// SYMA: A is symmetric with one scale per block (square digit blocks): its
// tiles are read from the upper triangle only, K-major where the 64-byte K
// stage lies at or left of the tile's rows and MN-major (mapA2, the same
// planes as 64 x 64 boxes) where it lies to the right: half the DRAM reads of
// A for products that stream it (the Chebyshev filter's G Y).
template <bool SYM, bool AMN, bool RESID, int BN = kBN, int NL = kS, bool SYMA = false>
__global__ void __launch_bounds__(kThreads, 1)
    ozaki_mma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     const __grid_constant__ CUtensorMap mapA2, const OzParams P, int64_t items) {
    static_assert(NL * BN <= 512 && BN % 16 == 0 && (BN / 2) % 8 == 0 && NL >= 1 && NL <= kSmax, "tile shape");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_TILE = kBM * kBK, B_TILE = BN * kBK;
    constexpr int STAGE = NL * (A_TILE + B_TILE);  // the NL digit tiles of A, then of B
    constexpr int STAGE_TX = STAGE;
    constexpr int STG = stages_for(BN, NL);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + STG * STAGE);
    uint64_t* empty = full + STG;
    uint64_t* tfull = empty + STG;
    uint64_t* tempty = tfull + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STG; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        bar_init(tfull, 1);
        bar_init(tempty, kEpiWarps);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tslot);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tslot;
    const int nkc = (int)(P.KCp / kBK);  // stages per digit block
    const int64_t per = P.per;

    if (warp == 0) {
        if (elect_one()) {
            int64_t g = 0;  // stage counter across items
            for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
                int64_t ob, mb, nb;
                decode_item<SYM, BN>(P, item, ob, mb, nb);
                for (int64_t gl = 0; gl < per * nkc; ++gl, ++g) {
                    const int st = (int)(g % STG);
                    bar_wait(&empty[st], (uint32_t)(((g / STG) & 1) ^ 1));
                    bar_expect_tx(&full[st], STAGE_TX);
                    const int64_t blk = ob * per + gl / nkc;
                    const int kx = (int)(gl % nkc) * kBK;
                    uint8_t* sa = base + st * STAGE;
                    uint8_t* sb = sa + NL * A_TILE;
                    const bool mn = SYMA && kx >= mb * kBM + kBM;  // stage right of the tile: read transposed
#pragma unroll
                    for (int s = 0; s < NL; ++s) {
                        const int plane = (int)(blk * P.nd + s);
                        if (SYMA && mn) {
                            tma_load_3d(sa + s * A_TILE, &mapA2, &full[st], (int)(mb * kBM), kx, plane);
                            tma_load_3d(sa + s * A_TILE + 4096, &mapA2, &full[st], (int)(mb * kBM + 64), kx, plane);
                        } else if (AMN) {
                            tma_load_3d(sa + s * A_TILE, &mapA, &full[st], (int)(mb * kBM), kx, plane);
                            tma_load_3d(sa + s * A_TILE + 4096, &mapA, &full[st], (int)(mb * kBM + 64), kx, plane);
                        } else {
                            tma_load_3d(sa + s * A_TILE, &mapA, &full[st], kx, (int)(mb * kBM), plane);
                        }
                        tma_load_3d(sb + s * B_TILE, &mapB, &full[st], kx, (int)(nb * BN), plane);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // signed digits, S32 accumulate; A MN-major for AMN. The B digit tiles
        // sit back to back in shared memory (one 80-row K-major matrix per
        // digit, same 512-byte atom stride), so digit i of A meets up to three
        // consecutive B digits j0..j0+2 in one MMA of N = 80 (j1 - j0 + 1): its
        // columns land exactly on the level accumulators i+j0 .. i+j1. 10 MMAs
        // per 32-byte k-slice instead of 21, each A tile read from shared memory
        // once per 240 columns instead of once per 80.
        constexpr uint32_t kAmn = AMN ? (1u << 15) : 0u;
        constexpr uint32_t kIdesc1 = idesc_i8<kBM, BN>() | kAmn;
        constexpr uint32_t kIdesc2 = idesc_i8<kBM, 2 * BN>() | kAmn;
        constexpr uint32_t kIdesc3 = idesc_i8<kBM, (3 * BN <= 256 ? 3 : 1) * BN>() | kAmn;
        constexpr int kGrp = 3 * BN <= 256 ? 3 : 2;  // UMMA N <= 256
        int64_t g = 0, cg = 0;  // stage and digit-block counters across items
        for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
            int64_t mb_item = 0;
            if (SYMA) {
                int64_t ob_, nb_;
                decode_item<SYM, BN>(P, item, ob_, mb_item, nb_);
            }
            for (int64_t cc = 0; cc < per; ++cc, ++cg) {
                if (cg > 0) {  // the epilogue has drained the previous block's levels
                    bar_wait(tempty, (uint32_t)((cg - 1) & 1));
                    fence_after_sync();
                }
                for (int kb = 0; kb < nkc; ++kb, ++g) {
                    const int st = (int)(g % STG);
                    bar_wait(&full[st], (uint32_t)((g / STG) & 1));
                    fence_after_sync();
                    if (elect_one()) {
                        const uint8_t* sa = base + st * STAGE;
                        const uint8_t* sb = sa + NL * A_TILE;
                        const bool mn = SYMA && (int64_t)kb * kBK >= mb_item * kBM + kBM;
                        const uint32_t amn = (AMN || mn) ? (1u << 15) : 0u;
#pragma unroll
                        for (int kk = 0; kk < kBK / 32; ++kk) {
                            // digit 1 of A spans every level: its MMAs start the block
                            const uint32_t acc0 = (kb > 0 || kk > 0) ? 1u : 0u;
#pragma unroll
                            for (int i = 1; i <= NL; ++i) {
                                const uint64_t da = (AMN || mn) ? sdesc_mn_sw64(sa + (i - 1) * A_TILE + kk * 2048, 4096)
                                                                : sdesc_k_sw64(sa + (i - 1) * A_TILE) + (uint64_t)(kk * 2);
                                const int jmax = NL + 1 - i;  // levels i + j <= NL + 1
#pragma unroll
                                for (int j0 = 1; j0 <= jmax; j0 += kGrp) {
                                    const int nj = jmax - j0 + 1 < kGrp ? jmax - j0 + 1 : kGrp;
                                    const uint32_t idesc = (nj == 3 ? kIdesc3 : (nj == 2 ? kIdesc2 : kIdesc1)) | amn;
                                    const uint64_t db = sdesc_k_sw64(sb + (j0 - 1) * B_TILE) + (uint64_t)(kk * 2);
                                    mma_i8(tmem + (uint32_t)((i + j0 - 2) * BN), da, db, idesc, i == 1 ? acc0 : 1u);
                                }
                            }
                        }
                        mma_commit(&empty[st]);
                    }
                    __syncwarp();
                }
                if (elect_one()) mma_commit(tfull);
                __syncwarp();
            }
        }
    } else {
        // epilogue: warp w drains TMEM lanes 32*(w%4) .. +32 (rows of the
        // tile), columns [h*40, h*40 + 40) with h = (w - 2) / 4
        const int q = warp & 3, h = (warp - 2) >> 2;
        constexpr int NH = BN / 2;
        int64_t cg = 0;
        double rsd = 0.0, rsx = 0.0;  // RESID: this thread's residual sums
        for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
            int64_t ob, mb, nb;
            decode_item<SYM, BN>(P, item, ob, mb, nb);
            const int64_t m = mb * kBM + q * 32 + lane;
            const int64_t n0 = nb * BN + h * NH;
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * NH);
            if constexpr (!SYM) {
                // one digit block per item (per == 1): each 8-column chunk goes
                // straight from TMEM to C (or into the residual sums)
                const bool xrow = RESID && m < P.M && ob * P.M + m < P.m_total;
                double xv[RESID ? NH : 1];
                if constexpr (RESID) {  // X loads in flight while the MMAs run
                    const double* X = P.X + ob * P.strideX + m;
#pragma unroll
                    for (int j = 0; j < NH; ++j) xv[j] = xrow && n0 + j < P.N ? __ldcs(X + (n0 + j) * P.ldx) : 0.0;
                }
                // fused Chebyshev step: b Y + c Yp in flight while the MMAs run
                constexpr bool kCheb = SYMA && !RESID;
                double pre[kCheb ? NH : 1];
                double ca = 1.0;
                const bool cheb = kCheb && P.cy != nullptr;
                if constexpr (kCheb) {
                    if (cheb) {
                        const double* cf = P.ccoef + 3 * ob;
                        ca = cf[0];
                        const double cb = cf[1], cc = cf[2];
                        const bool row = m < P.M;
                        const double* y = P.cy + ob * P.strideC + m;
                        const double* yp = P.cyp + ob * P.strideC + m;
                        // 16 loads in flight per round (the first use of a load
                        // waits for it: four DRAM round trips, not NH)
#pragma unroll
                        for (int c8 = 0; c8 < NH; c8 += 8) {
                            double ya[8], yb[8];
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj) {
                                const int64_t n = n0 + c8 + jj;
                                const bool ok = row && n < P.N;
                                ya[jj] = ok ? __ldcs(y + n * P.ldc) : 0.0;
                                yb[jj] = ok && cc != 0.0 ? __ldcs(yp + n * P.ldc) : 0.0;
                            }
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj) pre[c8 + jj] = fma(cc, yb[jj], cb * ya[jj]);
                        }
                    }
                }
                bar_wait(tfull, (uint32_t)(cg & 1));
                fence_after_sync();
                const double sm = m < P.M ? (P.sa ? P.sa[ob * P.M + m] : 1.0) : 0.0;
                const double* sc = P.sb + ob * P.N;
                double* C = RESID ? nullptr : P.C + ob * P.strideC;
#pragma unroll
                for (int c = 0; c < NH / 8; ++c) {  // all six levels of 8 columns in flight
                    int32_t v[NL][8];
#pragma unroll
                    for (int l = 0; l < NL; ++l) tmem_ld_32x32b_x8(ta + (uint32_t)(l * BN + c * 8), v[l]);
                    tmem_ld_wait();
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const int j = c * 8 + jj;
                        const int64_t n = n0 + j;
                        double inner = 0.0;
#pragma unroll
                        for (int l = NL - 1; l >= 0; --l)  // smallest weight first
                            inner = fma((double)v[l][jj], ldexp(1.0, -14 - 8 * l), inner);
                        const double val = (inner * sm) * (n < P.N ? sc[n] : 0.0);
                        if constexpr (RESID) {  // columns past N: x = val = 0
                            const double r = xv[j] - val;
                            rsd = fma(r, r, rsd);
                            rsx = fma(xv[j], xv[j], rsx);
                        } else if (m < P.M && n < P.N && (P.m_total == 0 || ob * P.M + m < P.m_total)) {
                            if constexpr (kCheb)
                                C[m + n * P.ldc] = cheb ? fma(ca, val, pre[j]) : val;
                            else
                                C[m + n * P.ldc] = val;  // (m, n), coalesced over the warp's rows
                        }
                    }
                }
                fence_before_sync();
                __syncwarp();
                if (lane == 0) bar_arrive(tempty);  // the MMAs may overwrite the levels
                ++cg;
            } else {
                double acc[NH];
#pragma unroll
                for (int j = 0; j < NH; ++j) acc[j] = 0.0;
                for (int64_t cc = 0; cc < per; ++cc, ++cg) {
                    bar_wait(tfull, (uint32_t)(cg & 1));
                    fence_after_sync();
                    const int64_t blk = ob * per + cc;
                    const double sm = m < P.M ? P.sa[blk * P.M + m] : 0.0;
                    const double* sc = P.sb + blk * P.N;
#pragma unroll
                    for (int c = 0; c < NH / 8; ++c) {
                        int32_t v[NL][8];
#pragma unroll
                        for (int l = 0; l < NL; ++l) tmem_ld_32x32b_x8(ta + (uint32_t)(l * BN + c * 8), v[l]);
                        tmem_ld_wait();
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            const int j = c * 8 + jj;
                            const int64_t n = n0 + j;
                            double inner = 0.0;
#pragma unroll
                            for (int l = NL - 1; l >= 0; --l)
                                inner = fma((double)v[l][jj], ldexp(1.0, -14 - 8 * l), inner);
                            // the diagonal of a Gram from the FP64 sums of squares: its
                            // dropped same-digit pair products are squares (biased > 0)
                            if (n == m)
                                acc[j] += P.sq[blk * P.M + m];
                            else
                                acc[j] = fma(inner * sm, n < P.N ? sc[n] : 0.0, acc[j]);
                        }
                    }
                    fence_before_sync();
                    __syncwarp();
                    if (lane == 0) bar_arrive(tempty);
                }
                if (m < P.M) {
                    double* C = P.C + ob * P.strideC;
                    // the mirror (n, m) holds the same exact integer sums. A lane owns
                    // row m, so its mirrored values are contiguous along n: four at a
                    // time as one 32-byte store (a full sector per lane) when the
                    // output is 32-byte aligned; one value at a time (a quarter sector
                    // per lane per store) measured 0.6-1.2 ms of the 11 ms cfg5 slice
                    // Grams
                    const bool v4 = (P.ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(C) & 31) == 0;
#pragma unroll
                    for (int j = 0; j < NH; j += 4) {  // fully unrolled: acc stays in registers
                        const int64_t n = n0 + j;
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (n + q < P.N) C[m + (n + q) * P.ldc] = acc[j + q];  // (m, n), coalesced over the warp's rows
                        double* mp = C + n + m * P.ldc;
                        if (v4 && n + 3 < P.N) {
                            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(mp), "d"(acc[j]),
                                         "d"(acc[j + 1]), "d"(acc[j + 2]), "d"(acc[j + 3])
                                         : "memory");
                        } else {
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                if (n + q < P.N) mp[q] = acc[j + q];
                        }
                    }
                }
            }
        }
        if (RESID) {  // fixed-order warp sums -> shared memory
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                rsd += __shfl_xor_sync(0xffffffffu, rsd, o);
                rsx += __shfl_xor_sync(0xffffffffu, rsx, o);
            }
            if (lane == 0) {
                reinterpret_cast<double*>(tslot + 2)[2 * (warp - 2)] = rsd;
                reinterpret_cast<double*>(tslot + 2)[2 * (warp - 2) + 1] = rsx;
            }
        }
    }
    fence_before_sync();
    __syncthreads();
    if (RESID && threadIdx.x == 0) {  // fixed-order CTA sum of the epilogue warps
        const double* ws = reinterpret_cast<const double*>(tslot + 2);
        double sd = 0.0, sx = 0.0;
        for (int w = 0; w < kEpiWarps; ++w) {
            sd += ws[2 * w];
            sx += ws[2 * w + 1];
        }
        P.partial[2 * blockIdx.x] = sd;
        P.partial[2 * blockIdx.x + 1] = sx;
    }
    if (warp == 1) tmem_free<512>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 3-D uint8 map over the digit planes: (k, row, plane), box (kBK, rows, 1),
// SWIZZLE_64B (rows beyond `cols` read as zeros: they never reach another plane).
bool make_digit_map(CUtensorMap* map, const int8_t* D, int64_t KCp, int64_t cols, int64_t planes, int box_rows) {
    HostProf hp_("make_digit_map");
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)KCp, (cuuint64_t)cols, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)KCp, (cuuint64_t)(KCp * cols)};
    cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(D), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

std::atomic<int> g_ozaki{-1};
bool ozaki_enabled() {
    int v = g_ozaki.load();
    if (v < 0) {
        const char* e = std::getenv("PPC_OZAKI");
        v = (e && e[0] == '0') ? 0 : 1;
        g_ozaki.store(v);
    }
    return v == 1;
}

// Digit levels of the data-driven Q's Gram SYRK (PPC_GRAM_LEVELS = 5 or 6,
// default 6). Five levels (15 digit pairs, levels 2..6) drop the level-7
// pair products, each <= 2^-40 sigma_a sigma_b per row with balanced signs:
// over a K-row chunk they add ~2^-41.6 sqrt(6 K) sigma_a sigma_b. Measured
// (cfg5): the step 127 -> 121 ms (the SYRK is not purely tensor-bound, so
// 15/21 of the pairs save less than 15/21 of its time), with the Gram 256x
// further from FP64 (i.i.d. Gaussian 2^18 x 512: 5e-13 of max|G| instead of
// ~2e-15). Kept as an A/B switch; the default stays at FP64-level accuracy.
// Sub-chunks per Gram plan chunk (PPC_GRAM_SUB, default 4; 1 = off); must
// divide the chunk's 4096-row block count.
int64_t gram_subchunks(int64_t per) {
    static const int64_t v = std::getenv("PPC_GRAM_SUB") ? std::atoll(std::getenv("PPC_GRAM_SUB")) : 4;
    return (v > 1 && per % v == 0) ? v : 1;
}

// out[g][e] = sum_{u < n} in[g n + u][e] in u order (fixed)
__global__ void sum_groups_kernel(const double* __restrict__ in, int64_t n, int64_t elems, int64_t total,
                                  double* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t g = i / elems, e = i - g * elems;
        const double* p = in + g * n * elems + e;
        double v = p[0];
        for (int64_t u = 1; u < n; ++u) v += p[u * elems];
        out[i] = v;
    }
}

int gram_levels() {
    static const int v = (std::getenv("PPC_GRAM_LEVELS") && std::atoi(std::getenv("PPC_GRAM_LEVELS")) == 5) ? 5 : kS;
    return v;
}

int64_t ozaki_grid(int64_t items) { return std::min<int64_t>(items, ctx().sms); }  // one persistent CTA per SM

template <bool SYM, bool AMN = false, bool RESID = false, int BN = kBN, int NL = kS, bool SYMA = false>
void launch_mma(const CUtensorMap& ma, const CUtensorMap& mb, const OzParams& P, int64_t items, cudaStream_t s,
                const CUtensorMap* ma2 = nullptr) {
    // stages + barriers + TMEM slot + the epilogue warps' residual sums
    constexpr int STG = stages_for(BN, NL);
    const size_t smem = 1024 + (size_t)STG * NL * (kBM + BN) * kBK + (2 * STG + 2) * 8 + 16 + 16 * kEpiWarps;
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, [&] {
        PPC_CUDA_CHECK(cudaFuncSetAttribute(ozaki_mma_kernel<SYM, AMN, RESID, BN, NL, SYMA>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    if (items == 0) return;
    ozaki_mma_kernel<SYM, AMN, RESID, BN, NL, SYMA><<<(unsigned)ozaki_grid(items), kThreads, smem, s>>>(
        ma, mb, ma2 ? *ma2 : ma, P, items);
    count_launch();
    check_launch("ozaki_mma");
}

int64_t tri_tiles(int64_t n, int64_t bn = kBN) {
    const int64_t mtiles = (n + kBM - 1) / kBM;
    int64_t tiles = 0;
    for (int64_t nb = 0; nb < (n + bn - 1) / bn; ++nb)
        tiles += std::min<int64_t>((nb * bn + bn - 1) / kBM + 1, mtiles);
    return tiles;
}

// Grams of `nout` outputs, each summing `per` digit blocks of d: out[ob] =
// sum over its blocks of X_blk^T X_blk (cols x cols, column-major).
void ozaki_syrk(const OzakiDigits& d, int64_t nout, int64_t per, double* out, cudaStream_t s, const char* stage,
                double rows_total, int64_t block_base = 0, int levels = kS) {
    // the nout * per blocks from block_base on
    const int8_t* D0 = d.D.as<int8_t>() + (size_t)block_base * d.nd * d.cols * d.KCp;
    // output tile width: 80 (6 x 80 TMEM columns, 2 ring stages) or 64
    // (3 stages; PPC_SYRK_BN=64)
    static const int bn = (std::getenv("PPC_SYRK_BN") && std::atoi(std::getenv("PPC_SYRK_BN")) == 64) ? 64 : kBN;
    CUtensorMap ma, mb;
    if (!make_digit_map(&ma, D0, d.KCp, d.cols, nout * per * d.nd, kBM) ||
        !make_digit_map(&mb, D0, d.KCp, d.cols, nout * per * d.nd, bn))
        fail(PPC_CUDA, "ozaki: tensor map encoding failed");
    OzParams P;
    P.M = P.N = d.cols;
    P.mtiles = (d.cols + kBM - 1) / kBM;
    P.tiles = tri_tiles(d.cols, bn);
    P.KCp = d.KCp;
    P.per = per;
    P.nd = d.nd;
    P.zmap = nullptr;
    P.sa = P.sb = d.sc.d() + block_base * d.cols;
    P.sq = d.sq.d() + block_base * d.cols;
    P.C = out;
    P.ldc = d.cols;
    P.strideC = d.cols * d.cols;
    P.X = nullptr;
    P.ldx = P.strideX = P.m_total = 0;
    P.partial = nullptr;
    // int8 ops of the levels (levels + 1) / 2 digit-pair products over the upper triangle
    StageTimer tk(stage, s, 2.0 * levels * (levels + 1) / 2 * rows_total * d.cols * d.cols / 2,
                  (double)levels * rows_total * d.cols);
    if (bn == 64)
        launch_mma<true, false, false, 64>(ma, mb, P, nout * P.tiles, s);
    else if (levels == 5)
        launch_mma<true, false, false, kBN, 5>(ma, mb, P, nout * P.tiles, s);
    else
        launch_mma<true>(ma, mb, P, nout * P.tiles, s);
}

}  // namespace

void OzakiDigits::split(const double* X, int64_t ldx, int64_t stride, int64_t rows_, int64_t cols_, int64_t KC,
                        int64_t nblk_, cudaStream_t s, const int* zmap, int64_t nz, int64_t chunk, int64_t per,
                        int* nonfinite, int ndig, int64_t block_base, int64_t alloc_blocks,
                        const double* fixed_max, int nwrite, bool trans_src, const double* rowscale) {
    HostProf hp_("ozaki_split");
    if (rowscale && (!stride || trans_src)) fail(PPC_ARGUMENT, "ozaki split: row scales need batched, untransposed blocks");
    if (trans_src && !stride) fail(PPC_ARGUMENT, "ozaki split: a transposed source needs batched blocks");
    if (ndig != kS && ndig != kSmax) fail(PPC_ARGUMENT, "ozaki split: 6 or 7 digits");
    if (block_base < 0 || (block_base > 0 && block_base + nblk_ > alloc_blocks))
        fail(PPC_ARGUMENT, "ozaki split: block range outside the allocation");
    nd = ndig;
    if (KC < 1 || KC > kKC) fail(PPC_ARGUMENT, "ozaki split: block length out of range");
    if (zmap && !stride) fail(PPC_ARGUMENT, "ozaki split: a block map needs batched blocks");
    rows = rows_;
    cols = cols_;
    const int64_t ncall = nblk_;
    nblk = std::max(nblk_, alloc_blocks);
    KCp = (KC + kBK - 1) / kBK * kBK;
    const size_t dbytes = sizeof(int8_t) * nblk * nd * cols * KCp, sbytes = sizeof(double) * nblk * cols;
    if (D.bytes() < dbytes) D = DeviceBuffer(dbytes);
    if (sc.bytes() < sbytes) sc = DeviceBuffer(sbytes);
    if (sq.bytes() < sbytes) sq = DeviceBuffer(sbytes);
    const int64_t launched = zmap ? nz : ncall;
    if (launched <= 0) return;
    const double total_rows = stride ? (double)std::min(KC, rows) * launched : (double)rows;
    StageTimer ts("ozaki_split", s, 0.0,
                  8.0 * total_rows * cols + (double)((nwrite > 0 && nwrite < nd) ? nwrite : nd) * total_rows * cols);
    int8_t* D0 = D.as<int8_t>() + (size_t)block_base * nd * cols * KCp;
    double* sc0 = sc.d() + block_base * cols;
    double* sq0 = sq.d() + block_base * cols;
    // columns per CTA: as many KCp-long columns as fit the 4096-element stage
    const int cpb = KCp <= 512 ? 8 : (KCp <= 1024 ? 4 : (KCp <= 2048 ? 2 : 1));
    dim3 grid((unsigned)((cols + cpb - 1) / cpb), (unsigned)launched);
    const int64_t ch = chunk ? chunk : KC, pr = per ? per : 1;
    const int nw = (nwrite > 0 && nwrite < nd) ? nwrite : nd;  // leading planes written
#define PPC_SPLIT(ND_, CPB_)                                                                                         \
    do {                                                                                                             \
        if (trans_src)                                                                                               \
            ozaki_split_kernel<ND_, CPB_, true><<<grid, 256, 0, s>>>(X, ldx, stride, rows, cols, KC, KCp, ch, pr,    \
                                                                     D0, sc0, sq0, zmap, nonfinite, fixed_max, nw,  \
                                                                     nullptr);                                       \
        else                                                                                                         \
            ozaki_split_kernel<ND_, CPB_><<<grid, 256, 0, s>>>(X, ldx, stride, rows, cols, KC, KCp, ch, pr, D0, sc0, \
                                                               sq0, zmap, nonfinite, fixed_max, nw, rowscale);       \
    } while (0)
    if (nd == kSmax) {
        if (cpb == 8) PPC_SPLIT(kSmax, 8); else if (cpb == 4) PPC_SPLIT(kSmax, 4);
        else if (cpb == 2) PPC_SPLIT(kSmax, 2); else PPC_SPLIT(kSmax, 1);
    } else {
        if (cpb == 8) PPC_SPLIT(kS, 8); else if (cpb == 4) PPC_SPLIT(kS, 4);
        else if (cpb == 2) PPC_SPLIT(kS, 2); else PPC_SPLIT(kS, 1);
    }
#undef PPC_SPLIT
    count_launch();
    check_launch("ozaki_split");
}

void ozaki_gemm(const OzakiDigits& A, const OzakiDigits& B, int64_t nbatch, const int* zmap, double* C, int64_t ldc,
                int64_t strideC, cudaStream_t s, int levels, bool sym_a, const ChebFuse* cheb) {
    HostProf hp_("ozaki_gemm");
    if (A.KCp != B.KCp) fail(PPC_ARGUMENT, "ozaki_gemm: K mismatch");
    if (levels != kS && levels != 4 && levels != 3) fail(PPC_ARGUMENT, "ozaki_gemm: levels must be 6, 4 or 3");
    // 64-wide output tiles for panels of <= 64 columns (the 80-wide tile
    // would spend a fifth of the MMAs on zero rows)
    const int bn = (B.cols <= 64) ? 64 : kBN;
    if (levels != kS && bn != 64) fail(PPC_ARGUMENT, "ozaki_gemm: reduced levels need <= 64 columns");
    CUtensorMap ma, mb;
    if (A.nd != B.nd) fail(PPC_ARGUMENT, "ozaki_gemm: digit counts differ");
    if (!make_digit_map(&ma, A.D.as<int8_t>(), A.KCp, A.cols, A.nblk * A.nd, kBM) ||
        !make_digit_map(&mb, B.D.as<int8_t>(), B.KCp, B.cols, B.nblk * B.nd, bn))
        fail(PPC_CUDA, "ozaki: tensor map encoding failed");
    OzParams P;
    P.M = A.cols;
    P.N = B.cols;
    P.mtiles = (P.M + kBM - 1) / kBM;
    P.tiles = P.mtiles * ((P.N + bn - 1) / bn);
    P.KCp = A.KCp;
    P.per = 1;
    P.nd = A.nd;
    P.zmap = zmap;
    P.sa = A.sc.d();
    P.sb = B.sc.d();
    P.sq = nullptr;
    P.C = C;
    P.ldc = ldc;
    P.strideC = strideC;
    P.X = nullptr;
    P.ldx = P.strideX = P.m_total = 0;
    P.partial = nullptr;
    const double K = (double)std::min(A.rows, kKC);
    if (cheb) {
        if (!(sym_a && bn == 64 && A.cols == A.rows && A.KCp == A.cols && A.nd == kS))
            fail(PPC_ARGUMENT, "ozaki_gemm: the fused Chebyshev step needs a symmetric A");
        P.cy = cheb->Y;
        P.cyp = cheb->Yp;
        P.ccoef = cheb->coef;
    }
    StageTimer tk(levels == kS ? "ozaki_gemm" : (levels == 4 ? "ozaki_gemm_l4" : "ozaki_gemm_l3"), s,
                  2.0 * levels * (levels + 1) / 2 * (double)nbatch * P.M * P.N * K,
                  (double)levels * nbatch * (P.M + P.N) * K);
    if (sym_a && bn == 64 && A.cols == A.rows && A.KCp == A.cols && A.nd == kS) {
        CUtensorMap ma2;  // the same planes as 64 x 64 MN-major boxes
        if (!make_digit_map(&ma2, A.D.as<int8_t>(), A.KCp, A.cols, A.nblk * A.nd, 64))
            fail(PPC_CUDA, "ozaki: tensor map encoding failed");
        if (levels == kS) launch_mma<false, false, false, 64, kS, true>(ma, mb, P, nbatch * P.tiles, s, &ma2);
        else if (levels == 4) launch_mma<false, false, false, 64, 4, true>(ma, mb, P, nbatch * P.tiles, s, &ma2);
        else launch_mma<false, false, false, 64, 3, true>(ma, mb, P, nbatch * P.tiles, s, &ma2);
        return;
    }
    if (bn == kBN) launch_mma<false>(ma, mb, P, nbatch * P.tiles, s);
    else if (levels == kS) launch_mma<false, false, false, 64, kS>(ma, mb, P, nbatch * P.tiles, s);
    else if (levels == 4) launch_mma<false, false, false, 64, 4>(ma, mb, P, nbatch * P.tiles, s);
    else launch_mma<false, false, false, 64, 3>(ma, mb, P, nbatch * P.tiles, s);
}

bool ozaki_path_on() { return ozaki_enabled(); }

namespace {
// out[g] = max over blocks b and columns c of group g (c / group == g) of
// (sc/2) sqrt(K) / ||x||: sc/2 bounds max|x| from above (sc in (2, 4] max|x|),
// so this is >= the column's peak ratio max|x| sqrt(K) / ||x||_2 and < twice
// it; zero columns count 0. CTA (g, y) scans blocks y, y + gridDim.y, ... of
// group g (all loads of a thread issued before the max), one block-level
// max, one atomic max of the (non-negative) bit patterns per CTA:
// order-independent.
__global__ void __launch_bounds__(256) peak_ratio_kernel(const double* __restrict__ sc, const double* __restrict__ sq,
                                                         int64_t cols, int64_t nblk, double sqrtK, int64_t group,
                                                         unsigned long long* __restrict__ out) {
    const int64_t g = blockIdx.x;
    const int64_t c0 = g * group, c1 = std::min<int64_t>(c0 + group, cols), gw = c1 - c0;
    const int64_t n = gw * ((nblk - blockIdx.y + gridDim.y - 1) / gridDim.y);
    double mx = 0.0;
    for (int64_t e0 = threadIdx.x; e0 < n; e0 += 8 * blockDim.x) {
        double qv[8], sv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t e = e0 + u * blockDim.x;
            const int64_t b = blockIdx.y + (e / gw) * gridDim.y, c = c0 + e % gw;
            const bool ok = e < n;
            qv[u] = ok ? sq[b * cols + c] : 0.0;
            sv[u] = ok ? sc[b * cols + c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (!(qv[u] <= DBL_MAX && sv[u] <= DBL_MAX)) mx = INFINITY;  // NaN / inf in the block column: fail the gate
            else if (qv[u] > 0.0) mx = fmax(mx, 0.5 * sv[u] * sqrtK / sqrt(qv[u]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
        if (mx > 0.0) atomicMax(out + g, (unsigned long long)__double_as_longlong(mx));
    }
}
}  // namespace

int64_t ozaki_peak_groups(const OzakiDigits& d, int64_t group) { return (d.cols + group - 1) / group; }

void ozaki_peak_ratios_async(const OzakiDigits& d, int64_t K, int64_t group, double* out, cudaStream_t s) {
    const int64_t ng = ozaki_peak_groups(d, group);
    PPC_CUDA_CHECK(cudaMemsetAsync(out, 0, sizeof(double) * ng, s));  // +0.0
    const int64_t ny = std::max<int64_t>(1, std::min<int64_t>(d.nblk, (4 * 148 + ng - 1) / ng));
    peak_ratio_kernel<<<dim3((unsigned)ng, (unsigned)ny), 256, 0, s>>>(
        d.sc.d(), d.sq.d(), d.cols, d.nblk, std::sqrt((double)K), group, reinterpret_cast<unsigned long long*>(out));
    count_launch();
    check_launch("peak_ratio");
}

std::vector<double> ozaki_peak_ratios(const OzakiDigits& d, int64_t K, int64_t group, cudaStream_t s) {
    const int64_t ng = ozaki_peak_groups(d, group);
    std::vector<double> h((size_t)ng);
    DeviceBuffer out(sizeof(double) * ng);
    ozaki_peak_ratios_async(d, K, group, out.d(), s);
    PPC_CUDA_CHECK(cudaMemcpyAsync(h.data(), out.d(), sizeof(double) * ng, cudaMemcpyDeviceToHost, s));
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    return h;
}

bool ozaki_gram_eligible(int64_t n3, int64_t chunk) { return ozaki_enabled() && n3 >= 128 && chunk >= 4096; }

bool ozaki_gemm_eligible(int64_t M, int64_t K) { return ozaki_enabled() && M >= kBM && K >= 256 && K <= kKC; }

namespace {

// Bt[c] (p x n3, column-major) = diag(sigma_c) Q^T: the per-(row block,
// slice) scales of the core's digits folded into the transform.
__global__ void fold_qt_kernel(const double* __restrict__ sc, const double* __restrict__ Q, int64_t n3, int64_t p,
                               int64_t total, double* __restrict__ Bt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t c = i / (p * n3), r = i - c * p * n3, n = r % p, j = r / p;
        Bt[i] = sc[c * p + n] * Q[j + n * n3];
    }
}

}  // namespace

bool ozaki_recon_residual(const double* X, int64_t N, int64_t n3, const double* Ch, const double* Q, int64_t p,
                          double sums[2], cudaStream_t s) {
    if (!ozaki_enabled() || n3 < kBN || p < 32 || p > kKC || N < kKC) return false;
    const int64_t nblk = (N + kKC - 1) / kKC;
    // A = the core's digits per (4096-row block, slice), read MN-major
    OzakiDigits cd, bd;
    cd.split(Ch, N, 0, N, p, kKC, nblk, s, nullptr, 0, kKC, 1);
    DeviceBuffer bt(sizeof(double) * nblk * p * n3);
    {
        const int64_t total = nblk * p * n3;
        fold_qt_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(cd.sc.d(), Q, n3, p,
                                                                                               total, bt.d());
        count_launch();
        check_launch("fold_qt");
    }
    bd.split(bt.d(), p, p * n3, p, n3, p, nblk, s);
    CUtensorMap ma, mb;
    if (!make_digit_map(&ma, cd.D.as<int8_t>(), cd.KCp, p, nblk * cd.nd, 64) ||
        !make_digit_map(&mb, bd.D.as<int8_t>(), bd.KCp, n3, nblk * bd.nd, kBN))
        fail(PPC_CUDA, "ozaki: tensor map encoding failed");
    OzParams P;
    P.M = kKC;
    P.N = n3;
    P.mtiles = kKC / kBM;
    P.tiles = P.mtiles * ((n3 + kBN - 1) / kBN);
    P.KCp = bd.KCp;  // the K extent: p, padded
    P.per = 1;
    P.nd = cd.nd;
    P.zmap = nullptr;
    P.sa = nullptr;  // folded into Bt
    P.sb = bd.sc.d();
    P.sq = nullptr;
    P.C = nullptr;
    P.ldc = P.strideC = 0;
    P.X = X;
    P.ldx = N;
    P.strideX = kKC;
    P.m_total = N;
    const int64_t items = nblk * P.tiles, grid = ozaki_grid(items);
    DeviceBuffer part(sizeof(double) * 2 * (grid + 1));
    P.partial = part.d();
    {
        StageTimer tk("ozaki_resid", s, 2.0 * kS * (kS + 1) / 2 * (double)N * n3 * p, 8.0 * N * n3);
        launch_mma<false, true, true>(ma, mb, P, items, s);
    }
    double* fin = part.d() + 2 * grid;
    launch_reduce_pairs(part.d(), grid, fin, s);
    PPC_CUDA_CHECK(cudaMemcpyAsync(sums, fin, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    return true;
}

bool ozaki_gram_partials(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk, int64_t nchunks,
                         double* parts, cudaStream_t s, int* nonfinite, OzakiDigits* keep, int64_t block_base,
                         int64_t total_blocks) {
    if (!ozaki_enabled()) return false;
    // The integer path pays off once each output tile sees a long K range.
    // The decision depends on the plan (n3, chunk) only, never on this
    // call's row count: every row group of the host-streamed Gram and every
    // rank's shard takes the same path, so Q is bitwise the same for host and
    // device input and for 1..8 GPUs (gram_plan keeps chunks >= 4096 rows
    // whenever N >= 16384 with the path on).
    if (!ozaki_gram_eligible(n3, chunk)) return false;
    if (rows > chunk * nchunks) return false;
    // each plan chunk is split into ceil(chunk / 4096) blocks that never cross
    // a plan-chunk boundary, and its partial sums them in order inside one
    // work item: the partial does not depend on how the rows are sharded
    const int64_t per = (chunk + kKC - 1) / kKC;
    const int64_t nblk = nchunks * per;
    StageTimer tm("gram_ozaki", s, (double)rows * n3 * n3, 8.0 * rows * n3);
    const bool retain = keep && chunk % kKC == 0;
    OzakiDigits local;
    OzakiDigits& d = retain ? *keep : local;
    const int64_t base = retain ? block_base : 0;
    d.split(T, ldT, 0, rows, n3, kKC, nblk, s, nullptr, 0, chunk, per, nonfinite, retain ? kSmax : kS, base,
            retain ? total_blocks : 0);
    if (retain && base == 0 && total_blocks == 0) d.uniform = true;  // streamed groups: the caller decides
    // Each chunk's partial as nsub sub-chunk partials (per / nsub blocks each),
    // summed in sub-chunk order: the 62-odd tiles of a (sub-)chunk stream its
    // rows side by side, and the shorter work items keep them closer together
    // in K (better L2 reuse of the digit planes) and cut the last wave's idle
    // tail. The sum order depends on the plan only (sharding-invariant).
    const int64_t nsub = gram_subchunks(per);
    if (nsub > 1) {
        DeviceBuffer sub(sizeof(double) * nchunks * nsub * n3 * n3);
        ozaki_syrk(d, nchunks * nsub, per / nsub, sub.d(), s, "ozaki_syrk", (double)rows, base, gram_levels());
        const int64_t total = nchunks * n3 * n3;
        sum_groups_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(
            sub.d(), nsub, n3 * n3, total, parts);
        count_launch();
        check_launch("sum_groups");
    } else {
        ozaki_syrk(d, nchunks, per, parts, s, "ozaki_syrk", (double)rows, base, gram_levels());
    }
    return true;
}

bool ozaki_mode3_forward(const OzakiDigits& td, int64_t N, const double* Q, int64_t p, double* out, cudaStream_t s) {
    static const bool off = std::getenv("PPC_OZAKI_FWD") && std::getenv("PPC_OZAKI_FWD")[0] == '0';
    if (off || !ozaki_enabled() || !td.uniform || td.nd != kSmax || td.KCp != kKC) return false;
    const int64_t n3 = td.cols, nblk = std::min(td.nblk, (N + kKC - 1) / kKC);  // blocks holding rows < N
    if (p < 64 || p % 64 || n3 < 256 || n3 > kKC || nblk * kKC < N) return false;
    StageTimer tm("mode3_fwd", s, 2.0 * N * n3 * p, 8.0 * (N * n3 + N * p + n3 * p));
    // B_b = diag(sigma_b) Q per 4096-row block b of T (its column scales vary
    // along the contraction index, so they fold into Q's rows, not into the
    // epilogue): split straight from Q with the block's row scales (the 1 GB of
    // scaled copies at cfg5 used to be written by a fold kernel and read back)
    OzakiDigits bd;
    bd.split(Q, n3, n3 * p, n3, p, n3, nblk, s, nullptr, 0, 0, 0, nullptr, kSmax, 0, 0, nullptr, 0, false,
             td.sc.d());
    CUtensorMap ma, mb;
    if (!make_digit_map(&ma, td.D.as<int8_t>(), td.KCp, n3, nblk * td.nd, 64) ||
        !make_digit_map(&mb, bd.D.as<int8_t>(), bd.KCp, p, nblk * bd.nd, 64))
        fail(PPC_CUDA, "ozaki: tensor map encoding failed");
    OzParams P;
    P.M = kKC;
    P.N = p;
    P.mtiles = kKC / kBM;
    P.tiles = P.mtiles * (p / 64);
    P.KCp = bd.KCp;  // the K extent: n3
    P.per = 1;
    P.nd = kSmax;
    P.zmap = nullptr;
    P.sa = nullptr;  // folded into Bq
    P.sb = bd.sc.d();
    P.sq = nullptr;
    P.C = out;
    P.ldc = N;
    P.strideC = kKC;  // block b starts at row 4096 b
    P.X = nullptr;
    P.ldx = P.strideX = 0;
    P.m_total = N;    // rows past N in the last block are not stored
    P.partial = nullptr;
    {
        StageTimer tk("ozaki_fwd", s, 2.0 * kSmax * (kSmax + 1) / 2 * (double)N * n3 * p, (double)kSmax * N * n3);
        launch_mma<false, true, false, 64, kSmax>(ma, mb, P, nblk * P.tiles, s);
    }
    return true;
}

// --------------------------------------------- star product inverse transform
// C (M x N, leading dimension ldc) = A B with A (M x K) split row-wise (one
// power-of-two scale per row over its K <= 64 values) and B (K x N, N <= 256,
// a multiple of 32) split column-wise: the cfg4 inverse transform C^ x3 Q
// (K = p, N = n3). Rows are independent (any row blocking gives the same
// bits: the host pipeline and the row-sharded product equal the device call).
//
// Shape of the work: K is one 64-byte stage, so the generic persistent kernel
// (one TMEM accumulator set, register stores) serialized MMA and epilogue and
// lost to FP64 DMMA. Here B's digits stay resident in shared memory for the
// whole launch (6 planes x N x 64 B <= 96 KB), each 128-row tile's A digits
// take one 48 KB stage, the N columns run as 32-wide sub-tiles into two TMEM
// buffers (6 levels x 32 columns each), and the epilogue drains one buffer
// while the MMAs fill the other and streams every 128 x 32 FP64 sub-tile out
// with a TMA store from a double-buffered staging tile. The kernel is bound
// by the 8 bytes written per output: 2.1 GB at cfg4 in 0.58 ms, DRAM writes at
// 3.6 TB/s (about what a copy reaches in either direction). Direct st.global
// from the epilogue warps (16 column segments of 256 B per warp) took 1.0 ms.
namespace {

constexpr int kRgNB = 32;        // sub-tile width (output columns)
constexpr int kRgMaxSub = 8;     // N <= 256
constexpr int kRgEpiWarps = 8;   // two per TMEM lane quadrant (16 columns each)
constexpr int kRgThreads = (2 + kRgEpiWarps) * 32;

// Row-wise split: digit row j of D holds row j of X (rows x K <= 64,
// column-major, leading dimension ldx) scaled by sigma_j > 2 max_k |X(j, k)|
// (a power of two), cut into ND digits along k (D layout [plane][row][64],
// zero padded). CTA: 64 rows; warp w: rows 32 (w / 4) + lane (coalesced
// column loads), k in [16 (w % 4), +16); a row's values stay in registers
// between the max and the digits; the digits are staged in shared memory and
// written out as contiguous 64 x 64-byte runs per plane.
constexpr int kRowsPerSplit = 64;
template <int ND>
__global__ void __launch_bounds__(256) ozaki_split_rows_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows,
                                                               int K, int8_t* __restrict__ D,
                                                               double* __restrict__ scale) {
    constexpr int KCp = kBK, RS = KCp + 16;
    __shared__ __align__(16) uint8_t tile[ND * kRowsPerSplit * RS];
    __shared__ double rmx[4][kRowsPerSplit];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, half = w >> 2, kq = w & 3;
    const int64_t r0 = (int64_t)blockIdx.x * kRowsPerSplit;
    const int rl = half * 32 + lane;
    const int64_t row = r0 + rl;
    const bool live = row < rows;
    const double* x = X + (live ? row : 0);
    double v[16];
    double mx = 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const int k = 16 * kq + u;
        v[u] = (live && k < K) ? __ldg(x + (int64_t)k * ldx) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) mx = fmax(mx, fabs(v[u]) <= DBL_MAX ? fabs(v[u]) : INFINITY);  // NaN -> inf
    rmx[kq][rl] = mx;
    __syncthreads();
    mx = fmax(fmax(rmx[0][rl], rmx[1][rl]), fmax(rmx[2][rl], rmx[3][rl]));
    // a row holding a NaN or an infinity: zero digits and a NaN scale, the
    // mark star_inv_fixup_kernel recomputes the row by on FP64 FMAs
    const bool bad = !(mx <= DBL_MAX);
    if (bad) mx = 0.0;
    if (kq == 0 && live) scale[row] = bad ? NAN : (mx > 0.0 ? ldexp(1.0, ilogb(mx) + 2) : 0.0);
    const int e = mx > 0.0 ? ilogb(mx) + 2 : 0;
    constexpr int SH = 8 * (ND - 1);
    constexpr unsigned long long C80 = 0x8080808080808080ULL >> (64 - SH);
    const int e1 = (SH + 7 - e) / 2;
    const double scl1 = mx > 0.0 ? ldexp(1.0, e1) : 0.0, scl2 = ldexp(1.0, SH + 7 - e - e1);
#pragma unroll
    for (int u4 = 0; u4 < 4; ++u4) {
        uint32_t wd[ND];
#pragma unroll
        for (int t = 0; t < ND; ++t) wd[t] = 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long y = __double2ll_rn(v[4 * u4 + q] * scl1 * scl2);
            const long long U = y + (long long)C80;
            const uint64_t low = (uint64_t)U ^ C80;
            wd[0] |= (uint32_t)(uint8_t)(int8_t)(U >> SH) << (8 * q);
#pragma unroll
            for (int t = 1; t < ND; ++t) wd[t] |= (uint32_t)((low >> (SH - 8 * t)) & 0xFFu) << (8 * q);
        }
#pragma unroll
        for (int t = 0; t < ND; ++t)
            *reinterpret_cast<uint32_t*>(tile + ((size_t)t * kRowsPerSplit + rl) * RS + 16 * kq + 4 * u4) = wd[t];
    }
    __syncthreads();
    const int nr = (int)std::min<int64_t>(kRowsPerSplit, rows - r0);
    const int per_plane = nr * KCp / 16;
    for (int t = 0; t < ND; ++t) {
        uint4* dst = reinterpret_cast<uint4*>(D + ((size_t)t * rows + r0) * KCp);
        for (int c = threadIdx.x; c < per_plane; c += blockDim.x) {
            const int i = (c * 16) / KCp, b = (c * 16) % KCp;
            dst[c] = *reinterpret_cast<const uint4*>(tile + ((size_t)t * kRowsPerSplit + i) * RS + b);
        }
    }
}

struct RgParams {
    int64_t M;          // rows
    int N, nsub;        // columns, 32-wide sub-tiles
    int64_t tiles;      // 128-row tiles
    const double* sa;   // row scales [M]
    const double* sb;   // column scales [N]
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n)); }

__global__ void __launch_bounds__(kRgThreads, 1)
    ozaki_rowgemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                         const __grid_constant__ CUtensorMap mapC, const RgParams P) {
    constexpr int NL = kS;
    constexpr int A_PLANE = kBM * kBK;         // 8 KB
    constexpr int B_PLANE = kRgNB * kBK;       // 2 KB
    constexpr int STG_TILE = kRgNB * kBM * 8;  // 32 KB of FP64
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sB = base;                                            // [sub][plane] 2 KB each
    uint8_t* sA = sB + kRgMaxSub * NL * B_PLANE;                   // [plane] 8 KB each
    double* stg = reinterpret_cast<double*>(sA + NL * A_PLANE);    // 2 x [32 cols][128 rows]
    uint64_t* bfull = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg) + 2 * STG_TILE);
    uint64_t* afull = bfull + 1;
    uint64_t* aempty = afull + 1;
    uint64_t* tfull = aempty + 1;   // [2]
    uint64_t* tempty = tfull + 2;   // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
    __shared__ double sbs[kRgMaxSub * kRgNB];  // column scales x 2^-30
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int n = threadIdx.x; n < P.N; n += blockDim.x) sbs[n] = P.sb[n] * 0x1.0p-30;
    if (threadIdx.x == 0) {
        bar_init(bfull, 1);
        bar_init(afull, 1);
        bar_init(aempty, 1);
        for (int u = 0; u < 2; ++u) {
            bar_init(&tfull[u], 1);
            bar_init(&tempty[u], kRgEpiWarps);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tslot);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tslot;
    const int nsub = P.nsub;

    if (warp == 0) {
        if (elect_one()) {
            bar_expect_tx(bfull, (uint32_t)(nsub * NL * B_PLANE));
            for (int sb = 0; sb < nsub; ++sb)
                for (int t = 0; t < NL; ++t) tma_load_3d(sB + (sb * NL + t) * B_PLANE, &mapB, bfull, 0, sb * kRgNB, t);
            int64_t it = 0;
            for (int64_t tile = blockIdx.x; tile < P.tiles; tile += gridDim.x, ++it) {
                bar_wait(aempty, (uint32_t)((it & 1) ^ 1));
                bar_expect_tx(afull, (uint32_t)(NL * A_PLANE));
                for (int t = 0; t < NL; ++t) tma_load_3d(sA + t * A_PLANE, &mapA, afull, 0, (int)(tile * kBM), t);
            }
        }
    } else if (warp == 1) {
        bar_wait(bfull, 0u);
        int64_t it = 0, gs = 0;
        for (int64_t tile = blockIdx.x; tile < P.tiles; tile += gridDim.x, ++it) {
            bar_wait(afull, (uint32_t)(it & 1));
            fence_after_sync();
            for (int sb = 0; sb < nsub; ++sb, ++gs) {
                const int u = (int)(gs & 1);
                bar_wait(&tempty[u], (uint32_t)(((gs >> 1) & 1) ^ 1));
                fence_after_sync();
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < kBK / 32; ++kk) {
#pragma unroll
                        for (int i = 1; i <= NL; ++i) {
                            const uint64_t da = sdesc_k_sw64(sA + (i - 1) * A_PLANE) + (uint64_t)(kk * 2);
                            const int jmax = NL + 1 - i;
#pragma unroll
                            for (int j0 = 1; j0 <= jmax; j0 += 3) {
                                const int nj = jmax - j0 + 1 < 3 ? jmax - j0 + 1 : 3;
                                const uint32_t idesc = nj == 3 ? idesc_i8<kBM, 3 * kRgNB>()
                                                               : (nj == 2 ? idesc_i8<kBM, 2 * kRgNB>()
                                                                          : idesc_i8<kBM, kRgNB>());
                                const uint64_t db = sdesc_k_sw64(sB + (sb * NL + j0 - 1) * B_PLANE) + (uint64_t)(kk * 2);
                                mma_i8(tmem + (uint32_t)(u * NL * kRgNB + (i + j0 - 2) * kRgNB), da, db, idesc,
                                       (i == 1 && kk == 0) ? 0u : 1u);
                            }
                        }
                    }
                    mma_commit(&tfull[u]);
                }
                __syncwarp();
            }
            if (elect_one()) mma_commit(aempty);  // every MMA of the tile has read A
            __syncwarp();
        }
    } else {
        // warp w reads TMEM lanes 32 (w % 4) .. + 31 (the rows of the tile),
        // columns [16 h, 16 h + 16) of each sub-tile
        const int q = warp & 3, h = (warp - 2) >> 2;
        int64_t gs = 0;
        for (int64_t tile = blockIdx.x; tile < P.tiles; tile += gridDim.x) {
            const int64_t m = tile * kBM + q * 32 + lane;
            const double sm = m < P.M ? P.sa[m] : 0.0;
            for (int sb = 0; sb < nsub; ++sb, ++gs) {
                const int u = (int)(gs & 1);
                bar_wait(&tfull[u], (uint32_t)((gs >> 1) & 1));
                fence_after_sync();
                double* st = stg + (size_t)u * (kRgNB * kBM);
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(u * NL * kRgNB);
                // levels 0-2 and 3-5 combined exactly in 64-bit integers
                // (|v| < 2^31: |v0 2^16 + v1 2^8 + v2| < 2^48 converts to FP64
                // exactly), so each output costs two conversions and one FMA
                // instead of six of each: the FP64 pipe bounds this epilogue
                static_assert(NL == 6, "two three-level groups");
#pragma unroll
                for (int c = 2 * h; c < 2 * h + 2; ++c) {
                    int32_t v[NL][8];
#pragma unroll
                    for (int l = 0; l < NL; ++l) tmem_ld_32x32b_x8(ta + (uint32_t)(l * kRgNB + c * 8), v[l]);
                    tmem_ld_wait();
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const long long g0 = ((long long)v[0][jj] << 16) + ((long long)v[1][jj] << 8) + v[2][jj];
                        const long long g1 = ((long long)v[3][jj] << 16) + ((long long)v[4][jj] << 8) + v[5][jj];
                        // sum_l v_l 2^(-14-8l) = 2^-30 (g0 + 2^-24 g1); 2^-30 sits in sbs
                        const double t = fma((double)g1, 0x1.0p-24, (double)g0);
                        const double val = (t * sm) * sbs[sb * kRgNB + c * 8 + jj];  // broadcast read
                        asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(smem_u32(st + (c * 8 + jj) * kBM + q * 32 + lane)),
                                     "d"(val)
                                     : "memory");
                    }
                }
                fence_before_sync();
                __syncwarp();
                if (lane == 0) bar_arrive(&tempty[u]);  // the MMAs may refill this TMEM buffer
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                named_bar(1, kRgEpiWarps * 32);
                if (warp == 2 && lane == 0) {
                    asm volatile(
                        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                            &mapC),
                        "r"((int)(tile * kBM)), "r"(sb * kRgNB), "r"(0), "r"(smem_u32(st))
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                    // the other staging tile (stored one sub-tile ago) is read out
                    asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
                }
                named_bar(1, kRgEpiWarps * 32);
            }
        }
        if (warp == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 1) tmem_free<512>(tmem);
}

constexpr size_t rg_smem() {
    return 1024 + (size_t)kRgMaxSub * kS * kRgNB * kBK + (size_t)kS * kBM * kBK + 2 * (size_t)kRgNB * kBM * 8 + 8 * 8 +
           16;
}

// Bt (K x N) = alpha Q^T for Q (N x K, column-major): column n = alpha Q(n, :)
// Rows of the star inverse whose input holds a NaN or an infinity (scale
// marked NaN by the row split): C(r, :) = A(r, :) Bt on FP64 FMAs, so the
// non-finite pattern is the FP64 product's (its NaN / inf positions do not
// depend on the summation order). One warp per 32 scanned rows, lanes over
// the columns of each marked row.
__global__ void star_inv_fixup_kernel(const double* __restrict__ A, int64_t M, int K, const double* __restrict__ Bt,
                                      int N, const double* __restrict__ scale, double* __restrict__ C, int64_t ldc) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; r0 < M; r0 += warps * 32) {
        const int64_t r = r0 + lane;
        unsigned bad = __ballot_sync(0xffffffffu, r < M && isnan(scale[r]));
        while (bad) {
            const int b = __ffs(bad) - 1;
            bad &= bad - 1;
            const int64_t row = r0 + b;
            for (int c = lane; c < N; c += 32) {
                double acc = 0.0;
                for (int k = 0; k < K; ++k) acc = fma(A[row + (int64_t)k * M], Bt[k + (int64_t)c * K], acc);
                C[row + (int64_t)c * ldc] = acc;
            }
        }
    }
}

__global__ void star_bt_kernel(const double* __restrict__ Q, int64_t N, int64_t K, double alpha, double* __restrict__ Bt) {
    const int64_t total = K * N;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i % K, n = i / K;
        Bt[i] = alpha * Q[n + k * N];
    }
}

bool make_fp64_map(CUtensorMap* map, const double* X, int64_t M, int64_t N, int64_t ld, int bm, int bn) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)N, 1};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)ld * N * 8};
    cuuint32_t box[3] = {(cuuint32_t)bm, (cuuint32_t)bn, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (strides[0] % 16) return false;
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(X), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool ozaki_star_inverse_eligible(int64_t K, int64_t N) {
    static const bool off = std::getenv("PPC_OZAKI_STAR_INV") && std::getenv("PPC_OZAKI_STAR_INV")[0] == '0';
    return !off && ozaki_enabled() && K >= 32 && K <= kBK && N >= kRgNB && N <= kRgMaxSub * kRgNB && N % kRgNB == 0;
}

bool ozaki_star_inverse(const double* A, int64_t M, int64_t K, const double* Q, int64_t N, double alpha, double* C,
                        int64_t ldc, cudaStream_t s) {
    // (an odd ldc or a C not 16-byte aligned cannot carry the TMA store: FP64
    // DMMA then, for that call only)
    if (!ozaki_star_inverse_eligible(K, N) || M < 1 || (ldc & 1) || ldc < M ||
        (reinterpret_cast<uintptr_t>(C) & 15))
        return false;
    StageTimer tm("mode3_inv", s, 2.0 * M * K * N, 8.0 * (M * K + M * N + K * N));
    // A (M x K, leading dimension M): row-wise digits
    OzakiDigits ad;
    ad.nd = kS;
    ad.rows = K;
    ad.cols = M;
    ad.nblk = 1;
    ad.KCp = kBK;
    ad.D = DeviceBuffer(sizeof(int8_t) * kS * M * kBK);
    ad.sc = DeviceBuffer(sizeof(double) * M);
    {
        StageTimer ts("ozaki_split", s, 0.0, 8.0 * M * K + (double)kS * M * kBK);
        ozaki_split_rows_kernel<kS><<<(unsigned)((M + kRowsPerSplit - 1) / kRowsPerSplit), 256, 0, s>>>(
            A, M, M, (int)K, ad.D.as<int8_t>(), ad.sc.d());
        count_launch();
        check_launch("ozaki_split_rows");
    }
    // B = alpha Q^T (K x N): column-wise digits
    DeviceBuffer bt(sizeof(double) * K * N);
    star_bt_kernel<<<(unsigned)std::min<int64_t>((K * N + 255) / 256, 1024), 256, 0, s>>>(Q, N, K, alpha, bt.d());
    count_launch();
    check_launch("star_bt");
    OzakiDigits bd;
    bd.split(bt.d(), K, K * N, K, N, K, 1, s);
    CUtensorMap ma, mb, mc;
    if (!make_digit_map(&ma, ad.D.as<int8_t>(), kBK, M, kS, kBM) ||
        !make_digit_map(&mb, bd.D.as<int8_t>(), bd.KCp, N, bd.nd, kRgNB) || !make_fp64_map(&mc, C, M, N, ldc, kBM, kRgNB))
        fail(PPC_CUDA, "ozaki: tensor map encoding failed");
    RgParams P;
    P.M = M;
    P.N = (int)N;
    P.nsub = (int)(N / kRgNB);
    P.tiles = (M + kBM - 1) / kBM;
    P.sa = ad.sc.d();
    P.sb = bd.sc.d();
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, [] {
        PPC_CUDA_CHECK(cudaFuncSetAttribute(ozaki_rowgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)rg_smem()));
    });
    {
        // bytes: the FP64 output written and A's digit planes read (HBM-bound: 8 B per output)
        StageTimer tk("ozaki_star_inv", s, 2.0 * kS * (kS + 1) / 2 * (double)M * K * N,
                      8.0 * M * N + (double)kS * M * kBK);
        ozaki_rowgemm_kernel<<<(unsigned)std::min<int64_t>(P.tiles, ctx().sms), kRgThreads, rg_smem(), s>>>(ma, mb, mc,
                                                                                                          P);
        count_launch();
        check_launch("ozaki_rowgemm");
    }
    // non-finite rows (none in the common case: the kernel only scans the scales)
    star_inv_fixup_kernel<<<(unsigned)std::min<int64_t>((M + 255) / 256, 8 * (int64_t)ctx().sms), 256, 0, s>>>(
        A, M, (int)K, bt.d(), (int)N, ad.sc.d(), C, ldc);
    count_launch();
    check_launch("star_inv_fixup");
    return true;
}

bool ozaki_syrk_batched(const double* A, int64_t lda, int64_t strideA, int64_t rows, int64_t n, int64_t batch,
                        double* G, cudaStream_t s, int* nonfinite) {
    if (!ozaki_enabled()) return false;
    if (n < 128 || rows < 1024 || rows > kKC || batch < 1) return false;
    if (strideA < lda * n) return false;
    OzakiDigits d;
    d.split(A, lda, strideA, rows, n, rows, batch, s, nullptr, 0, 0, 0, nonfinite);
    ozaki_syrk(d, batch, 1, G, s, "ozaki_syrk_batched", (double)rows * batch);
    return true;
}

}  // namespace ppc

extern "C" int ppc_set_ozaki(int mode) {
    if (mode < 0 || mode > 1) return PPC_ARGUMENT;
    ppc::g_ozaki.store(mode);
    return 0;
}

extern "C" int ppc_get_ozaki(void) { return ppc::ozaki_path_on() ? 1 : 0; }

extern "C" int ppc_ozaki_syrk_batched(const double* A, int64_t lda, int64_t strideA, int64_t rows, int64_t n,
                                      int64_t batch, double* G) {
    return ppc::guarded([&] {
        if (!A || !G) ppc::fail(PPC_ARGUMENT, "null pointer");
        if (!ppc::ozaki_syrk_batched(A, lda, strideA, rows, n, batch, G, ppc::stream()))
            ppc::fail(PPC_ARGUMENT, "ozaki_syrk_batched: shape not eligible (or the path is off)");
    });
}
