// FP64 Gram SYRK on the INT8 tensor cores (tcgen05 kind::i8): the Ozaki
// scheme (Ozaki, Ogita, Oishi, Rump 2012; the INT8 form of Ootomo, Ozaki and
// Yokota 2024).
//
// The data-driven basis needs G = T^T T over N = n1*n2 pixel rows. Per chunk
// of KC rows and per column j of T, the column is scaled by a power of two
// sigma_j with |T(:,j)| / sigma_j <= 1/2 and cut into S signed 7-bit digits,
//     T(i,j) = sigma_j * ( sum_s d_s(i,j) 2^{-7s} + r(i,j) 2^{-7S} ),
// |d_s| <= 64, |r| <= 1/2 (every step is exact in FP64). Then
//     G(a,b) ~= sigma_a sigma_b sum_{L=2}^{S+1} 2^{-7L} Q_L(a,b),
//     Q_L = sum_{s+t=L} D_s^T D_t,
// where every Q_L is an exact int32 sum of int8 products (KC * 64^2 * S <
// 2^31) computed by tcgen05.mma into its own TMEM accumulator. The FP64
// epilogue adds the levels smallest first. With S = 7 the truncation is
// ~2^{-50} sigma_a sigma_b per product (sigma ~ the column max, so heavy-
// tailed columns lose relative precision on small entries: S = 6 measured
// 4e-12 of max|G| on the cfg5 CP data, S = 7 8e-15), the integer sums are
// exact, and the error does not grow with the chunk length.
//
// Kernels: ozaki_split_kernel (one CTA per (chunk, column): max, scale,
// digits), ozaki_syrk_kernel (TMA SWIZZLE_64B operand tiles of all S digit
// planes per stage, one elected thread issuing the S(S+1)/2 digit-pair MMAs,
// four epilogue warps draining TMEM), sub_sum_kernel (fixed-order sum of a
// plan chunk's sub-chunk partials).
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>

#include "internal.h"
#include "ozaki.h"
#include "umma_i8.cuh"

namespace ppc {

namespace {

using namespace umma;

constexpr int kS = 7;          // digits per value (49 bits; 6 digits measured 4e-12 of max|G| on cfg5-like data)
constexpr int kBM = 128;       // UMMA M
constexpr int kBN = 64;        // UMMA N (S levels x 64 columns of TMEM)
constexpr int kBK = 64;        // bytes (= int8 elements) of K per stage, SWIZZLE_64B
constexpr int kStages = 2;
constexpr int64_t kKC = 65536;  // rows per sub-chunk: 65536 * 64^2 * S < 2^31
// Tensor memory: S level accumulators (kBN columns each). Optionally (kATmem)
// the stage's A digit tiles are copied to TMEM after them and the MMAs read
// only B from shared memory; at S = 6 that measured no faster than reading
// both operands from shared memory, and at S = 7 it does not fit.
constexpr int kAcol = kS * kBN;
#ifndef PPC_OZAKI_ATMEM
#define PPC_OZAKI_ATMEM 0
#endif
constexpr bool kATmem = PPC_OZAKI_ATMEM;
static_assert(kAcol + (kATmem ? kS * (kBK / 32) * 8 : 0) <= 512, "TMEM budget");

// ------------------------------------------------------------------ split
// One CTA per (block c, column j): block c is rows [c*KC, c*KC+KC) of T
// (row sub-chunks, strideT = 0) or the whole of matrix T + c*strideT
// (batched). D layout: [(c*S + s)*n3 + j][KCp] int8. Blocks of up to
// kStageRows rows are read from HBM once (staged in shared memory for the
// digit pass); each thread emits four consecutive rows per digit as one
// 32-bit store.
constexpr int64_t kStageRows = 4096;  // 32 KB of shared memory (several CTAs per SM)

template <bool STAGE>
__global__ void __launch_bounds__(256) ozaki_split_kernel(const double* __restrict__ T, int64_t ldT, int64_t strideT,
                                                          int64_t rows, int64_t n3, int64_t KC, int64_t KCp,
                                                          int8_t* __restrict__ D, double* __restrict__ scale,
                                                          const int* __restrict__ zmap) {
    extern __shared__ double stage[];
    const int64_t j = blockIdx.x, c = zmap ? zmap[blockIdx.y] : blockIdx.y;
    const int64_t r0 = strideT ? 0 : c * KC;
    const int64_t len = std::max<int64_t>(0, std::min<int64_t>(KC, rows - r0));
    const double* col = T + (strideT ? c * strideT : 0) + j * ldT + r0;
    double mx = 0.0;
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
        const double v = col[i];
        if (STAGE) stage[i] = v;
        mx = fmax(mx, fabs(v));
    }
    __shared__ double red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        mx = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (threadIdx.x == 0) red[0] = mx;
    }
    __syncthreads();
    mx = red[0];
    // sigma = 2^e with mx / sigma <= 1/2 (mx = 0: all digits zero)
    const int e = mx > 0.0 ? ilogb(mx) + 2 : 0;
    if (threadIdx.x == 0) scale[c * n3 + j] = mx > 0.0 ? ldexp(1.0, e) : 0.0;
    int8_t* out = D + ((c * kS) * n3 + j) * KCp;
    const int64_t plane = n3 * KCp;
    for (int64_t i4 = (int64_t)threadIdx.x * 4; i4 < KCp; i4 += (int64_t)blockDim.x * 4) {
        uint32_t w[kS];
#pragma unroll
        for (int s = 0; s < kS; ++s) w[s] = 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t i = i4 + q;
            double x = i < len ? ldexp(STAGE ? stage[i] : col[i], -e) : 0.0;
#pragma unroll
            for (int s = 0; s < kS; ++s) {
                const double t = x * 128.0;
                const double d = rint(t);
                x = t - d;
                w[s] |= (uint32_t)(uint8_t)(int8_t)d << (8 * q);
            }
        }
#pragma unroll
        for (int s = 0; s < kS; ++s) *reinterpret_cast<uint32_t*>(out + s * plane + i4) = w[s];
    }
}

// ------------------------------------------------------------------- syrk
// One launch covers `items` = nbatch * tiles work items: item -> batch bi,
// tile t; bi -> operand/output block blk (zmap, else bi). SYM: the tiles are
// the upper triangle of an M x M Gram, written together with their mirror.
struct OzParams {
    int64_t M, N;          // output extents per block
    int64_t mtiles, tiles; // row tiles; tiles per block
    int64_t KCp;           // padded K length (multiple of kBK)
    const int* zmap;       // nullable batch -> block map
    const double* sa;      // row scales [blk][M]
    const double* sb;      // column scales [blk][N]
    double* C;             // output block blk at C + blk*strideC, (m, n) at m + n*ldc
    int64_t ldc, strideC;
};

// tile t (upper-triangle order) -> (mb, nb): column tile nb holds
// floor((nb*kBN + kBN - 1) / kBM) + 1 row tiles.
__device__ __forceinline__ void tri_tile(int64_t t, int64_t& mb, int64_t& nb) {
    nb = 0;
    for (;;) {
        const int64_t cnt = (nb * kBN + kBN - 1) / kBM + 1;
        if (t < cnt) break;
        t -= cnt;
        ++nb;
    }
    mb = t;
}

template <bool SYM>
__global__ void __launch_bounds__(192, 1)
    ozaki_mma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     const OzParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int A_TILE = kBM * kBK, B_TILE = kBN * kBK;
    constexpr int STAGE = kS * (A_TILE + B_TILE);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + kStages * STAGE);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t item = blockIdx.x;
    const int64_t bi = item / P.tiles;
    const int64_t sub = P.zmap ? P.zmap[bi] : bi;
    int64_t mb, nb;
    if (SYM) {
        tri_tile(item - bi * P.tiles, mb, nb);
    } else {
        const int64_t t = item - bi * P.tiles;
        mb = t % P.mtiles;
        nb = t / P.mtiles;
    }

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        bar_init(tfull, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tslot);
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = *tslot;
    const int nk = (int)(P.KCp / kBK);

    if (warp == 0) {
        if (elect_one()) {
            for (int kb = 0; kb < nk; ++kb) {
                const int st = kb % kStages;
                bar_wait(&empty[st], ((kb / kStages) & 1) ^ 1);
                bar_expect_tx(&full[st], STAGE);
                uint8_t* sa = base + st * STAGE;
                uint8_t* sb = sa + kS * A_TILE;
#pragma unroll
                for (int s = 0; s < kS; ++s) {
                    const int plane = (int)(sub * kS + s);
                    tma_load_3d(sa + s * A_TILE, &mapA, &full[st], kb * kBK, (int)(mb * kBM), plane);
                    tma_load_3d(sb + s * B_TILE, &mapB, &full[st], kb * kBK, (int)(nb * kBN), plane);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_i8<kBM, kBN>();
        for (int kb = 0; kb < nk; ++kb) {
            const int st = kb % kStages;
            bar_wait(&full[st], (kb / kStages) & 1);
            fence_after_sync();
            if (elect_one()) {
                const uint8_t* sa = base + st * STAGE;
                const uint8_t* sb = sa + kS * A_TILE;
                // A digit tiles -> TMEM (in issue order with the MMAs below and
                // after the previous stage's MMAs, which read the same columns)
#pragma unroll
                for (int s = 0; s < (kATmem ? kS : 0); ++s) {
                    const uint64_t da = sdesc_k_sw64(sa + s * A_TILE);
#pragma unroll
                    for (int kk = 0; kk < kBK / 32; ++kk)
                        tmem_cp_128x256b(tmem + (uint32_t)(kAcol + (s * (kBK / 32) + kk) * 8), da + (uint64_t)(kk * 2));
                }
#pragma unroll
                for (int l = 0; l < kS; ++l) {  // level L = l + 2
                    const int L = l + 2;
                    const int s_lo = L - kS > 1 ? L - kS : 1, s_hi = L - 1 < kS ? L - 1 : kS;
#pragma unroll
                    for (int s = s_lo; s <= s_hi; ++s) {
                        const int t = L - s;
                        const uint64_t db = sdesc_k_sw64(sb + (t - 1) * B_TILE);
#pragma unroll
                        for (int kk = 0; kk < kBK / 32; ++kk) {
                            const uint32_t acc = (kb > 0 || s > s_lo || kk > 0) ? 1u : 0u;
                            if (kATmem)
                                mma_i8_ts(tmem + (uint32_t)(l * kBN),
                                          tmem + (uint32_t)(kAcol + ((s - 1) * (kBK / 32) + kk) * 8),
                                          db + (uint64_t)(kk * 2), idesc, acc);
                            else
                                mma_i8(tmem + (uint32_t)(l * kBN), sdesc_k_sw64(sa + (s - 1) * A_TILE) + (uint64_t)(kk * 2),
                                       db + (uint64_t)(kk * 2), idesc, acc);
                        }
                    }
                }
                mma_commit(&empty[st]);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(tfull);
        __syncwarp();
    } else {
        // epilogue: warp w drains TMEM lanes 32*(w%4) .. +32 (rows of the tile)
        bar_wait(tfull, 0);
        fence_after_sync();
        const int q = warp & 3;
        const int64_t m = mb * kBM + q * 32 + lane;
        double acc[kBN];
#pragma unroll
        for (int j = 0; j < kBN; ++j) acc[j] = 0.0;
#pragma unroll 1
        for (int l = kS - 1; l >= 0; --l) {  // smallest weight first
            const double w = ldexp(1.0, -7 * (l + 2));
#pragma unroll
            for (int h = 0; h < kBN; h += 32) {
                int32_t v[32];
                tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(l * kBN + h), v);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[h + j] = fma((double)v[j], w, acc[h + j]);
            }
        }
        if (m < P.M) {
            const double sm = P.sa[sub * P.M + m];
            const double* sc = P.sb + sub * P.N;
            double* C = P.C + sub * P.strideC;
#pragma unroll 4
            for (int j = 0; j < kBN; ++j) {
                const int64_t n = nb * kBN + j;
                if (n >= P.N) break;
                const double v = acc[j] * sm * sc[n];
                C[m + n * P.ldc] = v;                // (m, n), coalesced over the warp's rows
                if (SYM) C[n + m * P.ldc] = v;       // mirror (n, m): the same exact integer sums
            }
        }
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 1) tmem_free<512>(tmem);
}

// parts[c] = sum_{u < per} sub[c*per + u] in ascending u (fixed order)
__global__ void sub_sum_kernel(const double* __restrict__ sub, int64_t per, int64_t elems, int64_t total,
                               double* __restrict__ parts) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t c = i / elems, e = i - c * elems;
        const double* p = sub + c * per * elems + e;
        double a = p[0];
        for (int64_t u = 1; u < per; ++u) a += p[u * elems];
        parts[i] = a;
    }
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

// 3-D int8 map over the digit planes: (k, row, plane), box (kBK, rows, 1),
// SWIZZLE_64B (rows beyond n3 read as zeros: they never reach another plane).
bool make_digit_map(CUtensorMap* map, const int8_t* D, int64_t KCp, int64_t n3, int64_t planes, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)KCp, (cuuint64_t)n3, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)KCp, (cuuint64_t)(KCp * n3)};
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

}  // namespace

void OzakiDigits::split(const double* X, int64_t ldx, int64_t stride, int64_t rows_, int64_t cols_, int64_t KC,
                        int64_t nblk_, cudaStream_t s, const int* zmap, int64_t nz) {
    rows = rows_;
    cols = cols_;
    nblk = nblk_;
    KCp = (KC + kBK - 1) / kBK * kBK;
    const size_t dbytes = sizeof(int8_t) * nblk * kS * cols * KCp, sbytes = sizeof(double) * nblk * cols;
    if (D.bytes() < dbytes) D = DeviceBuffer(dbytes);
    if (sc.bytes() < sbytes) sc = DeviceBuffer(sbytes);
    if (zmap && !stride) fail(PPC_ARGUMENT, "ozaki split: a block map needs batched blocks");
    const int64_t launched = zmap ? nz : nblk;
    if (launched <= 0) return;
    const double total_rows = stride ? (double)rows * launched : (double)rows;
    StageTimer ts("ozaki_split", s, 0.0, 8.0 * total_rows * cols + (double)kS * total_rows * cols);
    dim3 grid((unsigned)cols, (unsigned)launched);
    if (KC <= kStageRows) {
        const size_t sm = sizeof(double) * KC;
        static bool attr = false;
        if (!attr) {
            PPC_CUDA_CHECK(cudaFuncSetAttribute(ozaki_split_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)(sizeof(double) * kStageRows)));
            attr = true;
        }
        ozaki_split_kernel<true><<<grid, 256, sm, s>>>(X, ldx, stride, rows, cols, KC, KCp, D.as<int8_t>(), sc.d(),
                                                       zmap);
    } else {
        ozaki_split_kernel<false><<<grid, 256, 0, s>>>(X, ldx, stride, rows, cols, KC, KCp, D.as<int8_t>(), sc.d(),
                                                        zmap);
    }
    count_launch();
    check_launch("ozaki_split");
}

namespace {

template <bool SYM>
void launch_mma(const CUtensorMap& ma, const CUtensorMap& mb, const OzParams& P, int64_t items, cudaStream_t s) {
    const size_t smem = 1024 + (size_t)kStages * kS * (kBM + kBN) * kBK + (2 * kStages + 1) * 8 + 16;
    static bool attr = false;
    if (!attr) {
        PPC_CUDA_CHECK(cudaFuncSetAttribute(ozaki_mma_kernel<SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    if (items > 0x7fffffffLL) fail(PPC_ARGUMENT, "ozaki: too many tiles");
    if (items == 0) return;
    ozaki_mma_kernel<SYM><<<(unsigned)items, 192, smem, s>>>(ma, mb, P);
    count_launch();
    check_launch("ozaki_mma");
}

// Split + SYRK over nblk blocks of KC rows (see ozaki_split_kernel): out[c]
// (n3 x n3, column-major) = T_c^T T_c for every block c.
void ozaki_syrk_blocks(const double* T, int64_t ldT, int64_t strideT, int64_t rows, int64_t n3, int64_t KC,
                       int64_t nblk, double* out, cudaStream_t s, const char* stage) {
    OzakiDigits d;
    d.split(T, ldT, strideT, rows, n3, KC, nblk, s);
    CUtensorMap ma, mb;
    if (!make_digit_map(&ma, d.D.as<int8_t>(), d.KCp, n3, nblk * kS, kBM) ||
        !make_digit_map(&mb, d.D.as<int8_t>(), d.KCp, n3, nblk * kS, kBN))
        fail(PPC_CUDA, "ozaki: tensor map encoding failed");
    OzParams P;
    P.M = P.N = n3;
    P.mtiles = (n3 + kBM - 1) / kBM;
    P.tiles = 0;
    for (int64_t nb = 0; nb < (n3 + kBN - 1) / kBN; ++nb)
        P.tiles += std::min<int64_t>((nb * kBN + kBN - 1) / kBM + 1, P.mtiles);
    P.KCp = d.KCp;
    P.zmap = nullptr;
    P.sa = P.sb = d.sc.d();
    P.C = out;
    P.ldc = n3;
    P.strideC = n3 * n3;
    const double total_rows = strideT ? (double)rows * nblk : (double)rows;
    StageTimer tk(stage, s, 2.0 * kS * (kS + 1) / 2 * total_rows * n3 * n3 / 2, (double)kS * total_rows * n3);
    launch_mma<true>(ma, mb, P, nblk * P.tiles, s);
}

}  // namespace

void ozaki_gemm(const OzakiDigits& A, const OzakiDigits& B, int64_t nbatch, const int* zmap, double* C, int64_t ldc,
                int64_t strideC, cudaStream_t s) {
    if (A.KCp != B.KCp || A.rows != B.rows) fail(PPC_ARGUMENT, "ozaki_gemm: K mismatch");
    CUtensorMap ma, mb;
    if (!make_digit_map(&ma, A.D.as<int8_t>(), A.KCp, A.cols, A.nblk * kS, kBM) ||
        !make_digit_map(&mb, B.D.as<int8_t>(), B.KCp, B.cols, B.nblk * kS, kBN))
        fail(PPC_CUDA, "ozaki: tensor map encoding failed");
    OzParams P;
    P.M = A.cols;
    P.N = B.cols;
    P.mtiles = (P.M + kBM - 1) / kBM;
    P.tiles = P.mtiles * ((P.N + kBN - 1) / kBN);
    P.KCp = A.KCp;
    P.zmap = zmap;
    P.sa = A.sc.d();
    P.sb = B.sc.d();
    P.C = C;
    P.ldc = ldc;
    P.strideC = strideC;
    StageTimer tk("ozaki_gemm", s, 2.0 * kS * (kS + 1) / 2 * (double)nbatch * P.M * P.N * A.rows,
                  (double)kS * nbatch * (P.M + P.N) * A.rows);
    launch_mma<false>(ma, mb, P, nbatch * P.tiles, s);
}

bool ozaki_gemm_eligible(int64_t M, int64_t K) { return ozaki_enabled() && M >= kBM && K >= 256 && K <= kKC; }

bool ozaki_gram_partials(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk, int64_t nchunks,
                         double* parts, cudaStream_t s) {
    if (!ozaki_enabled()) return false;
    // the integer path pays off once each output tile sees a long K range
    if (n3 < 128 || n3 > 65535 || chunk < 4096 || rows < 4096 * 4) return false;
    if (rows > chunk * nchunks) return false;
    // sub-chunks of KC rows tile every plan chunk exactly (a longer plan
    // chunk must be a multiple of KC), so a plan chunk's partial never
    // depends on how the rows are sharded
    // (KC = kKC: longer sub-chunks keep the split's second read of each
    // column chunk L2-resident and the sub-chunk partials few; staging 16K-row
    // chunks in shared memory measured slower at one CTA per SM)
    if (chunk > kKC && chunk % kKC != 0) return false;
    const int64_t KC = std::min<int64_t>(chunk, kKC);
    const int64_t per_chunk = chunk / KC;
    const int64_t nsub = nchunks * per_chunk;
    if (nsub * kS > 65535) return false;
    StageTimer tm("gram_ozaki", s, (double)rows * n3 * n3, 8.0 * rows * n3);
    DeviceBuffer subp;
    double* out = parts;
    if (per_chunk > 1) {
        subp = DeviceBuffer(sizeof(double) * nsub * n3 * n3);
        out = subp.d();
    }
    ozaki_syrk_blocks(T, ldT, 0, rows, n3, KC, nsub, out, s, "ozaki_syrk");
    if (per_chunk > 1) {
        const int64_t elems = n3 * n3, total = nchunks * elems;
        sub_sum_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(out, per_chunk, elems,
                                                                                               total, parts);
        count_launch();
        check_launch("sub_sum");
    }
    return true;
}

bool ozaki_syrk_batched(const double* A, int64_t lda, int64_t strideA, int64_t rows, int64_t n, int64_t batch,
                        double* G, cudaStream_t s) {
    if (!ozaki_enabled()) return false;
    if (n < 128 || rows < 1024 || rows > kKC || batch < 1 || batch * kS > 65535) return false;
    if (strideA < lda * n) return false;
    ozaki_syrk_blocks(A, lda, strideA, rows, n, rows, batch, G, s, "ozaki_syrk_batched");
    return true;
}

}  // namespace ppc

extern "C" int ppc_set_ozaki(int mode) {
    if (mode < 0 || mode > 1) return PPC_ARGUMENT;
    ppc::g_ozaki.store(mode);
    return 0;
}
