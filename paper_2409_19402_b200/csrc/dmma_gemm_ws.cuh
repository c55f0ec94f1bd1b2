// Warp-specialized, persistent FP64 DMMA GEMM with TMA staging (sm_100a).
//
// Same math and shared-memory layout as dmma_gemm.cuh (32-byte interleaved
// quads -> conflict-free DMMA fragment reads), but:
//   - one producer warp issues cp.async.bulk.tensor (TMA) loads into an
//     S-stage ring guarded by mbarriers (full: tx-count; empty: one arrive
//     per consumer warp); consumers never __syncthreads in the main loop;
//   - CTAs are persistent (grid = #SMs) over a static tile schedule, so the
//     producer streams the next tile's operands while consumers run the
//     epilogue of the current one;
//   - the interleaved layout is expressed as a 5-D tensor map:
//       d0 = 4 (quad), d1 = other dim, d2 = contiguous-dim quads (within a
//       block), d3 = contiguous-dim blocks (k-blocked Gram layout), d4 = batch.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dmma_gemm.cuh"

namespace ppc {

struct WsParams {
    int64_t M, N, K;
    int64_t batch;
    int64_t mtiles, ntiles, tiles_per_batch, total_tiles;  // tile schedule
    int tri;     // symmetric: upper tiles only (mtiles == ntiles), mirrored store
    int nfast;   // raster
    int64_t kchunk;        // split-K: K range per split (tiles of different splits are distinct work items)
    int64_t splits;
    int64_t strideCsplit;
    double* C; int64_t ldc, strideC;
    const double* Cin; int64_t ldcin, strideCin;
    double alpha, beta;
    const double* X; int64_t ldx, strideX;  // RESID
    double* partial;                        // RESID: 2 per CTA
    int a_kblock, b_kblock;                 // log2 of the k-block (0 = none)
    const int* zmap;                        // nullable batch index indirection
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned addr = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT;\n"
        "}\n" ::"r"(addr),
        "r"(parity));
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
        "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// Tile coordinates of work item w (batch, split, m-tile, n-tile).
__device__ __forceinline__ void ws_tile(const WsParams& P, int64_t w, int64_t& b, int64_t& sp, int64_t& mt,
                                        int64_t& nt) {
    const int64_t per_split = P.tiles_per_batch;
    const int64_t per_batch = per_split * P.splits;
    b = w / per_batch;
    int64_t r = w - b * per_batch;
    if (P.zmap) b = P.zmap[b];
    int64_t t = r % per_split;
    sp = r / per_split;
    if (P.tri) {
        mt = 0;
        while (t >= P.ntiles - mt) {
            t -= P.ntiles - mt;
            ++mt;
        }
        nt = mt + t;
    } else if (P.nfast) {
        nt = t % P.ntiles;
        mt = t / P.ntiles;
    } else {
        mt = t % P.mtiles;
        nt = t / P.mtiles;
    }
}

// EPI_TSTORE: the plain store (beta = 0, no split, no mirror) through shared
// memory and a TMA bulk tensor store issued by a dedicated store warp, so the
// consumers start the next tile's MMAs while the previous tile drains to HBM
// (short-K products: the epilogue is a third of the tile's time otherwise).
enum { EPI_TSTORE = 2 };

template <int BM, int BN, int WARPS_M, int WARPS_N, int EPI>
constexpr int ws_threads() { return (WARPS_M * WARPS_N + 1 + (EPI == EPI_TSTORE ? 1 : 0)) * 32; }

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool AK, bool BNM, int EPI>
__global__ void __launch_bounds__(ws_threads<BM, BN, WARPS_M, WARPS_N, EPI>(), 1)
    dmma_gemm_ws_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                        const __grid_constant__ CUtensorMap mapX, const WsParams P) {
    constexpr int NCW = WARPS_M * WARPS_N;  // consumer warps
    constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
    constexpr int TM = WM / 8, TN = WN / 8;
    constexpr unsigned STAGE_BYTES = (BM * BK + BK * BN) * 8;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Bs = As + STAGES * BM * BK;
    // RESID: the tile's reference block X (BN columns of BM rows, [n][m])
    // is staged by TMA right after the operand ring; TSTORE: the output tile
    // ([n][m]) on its way to the TMA store
    constexpr bool XS = (EPI == EPI_RESID) || (EPI == EPI_TSTORE);
    double* Xs = Bs + STAGES * BK * BN;
    uint64_t* full = reinterpret_cast<uint64_t*>(Xs + (XS ? BM * BN : 0));
    uint64_t* empty = full + STAGES;
    uint64_t* xfull = empty + STAGES;
    uint64_t* xempty = xfull + 1;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        if constexpr (EPI == EPI_RESID) {
            mbar_init(xfull, 1);
            mbar_init(xempty, NCW);
        }
        if constexpr (EPI == EPI_TSTORE) {
            mbar_init(xfull, NCW);  // consumers wrote the tile
            mbar_init(xempty, 1);   // the store warp's TMA has read it
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();

    if constexpr (EPI == EPI_TSTORE) {
        if (warp == NCW + 1) {
            // -------------------------------------------- TMA store warp
            if (lane == 0) {
                asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mapX));
                unsigned ph = 0;
                for (int64_t w = blockIdx.x; w < P.total_tiles; w += gridDim.x) {
                    int64_t b, sp, mt, nt;
                    ws_tile(P, w, b, sp, mt, nt);
                    mbar_wait(xfull, ph);
                    asm volatile(
                        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                            &mapX),
                        "r"((int)(mt * BM)), "r"((int)(nt * BN)), "r"((int)b),
                        "r"((unsigned)__cvta_generic_to_shared(Xs))
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // Xs may be rewritten
                    mbar_arrive(xempty);
                    ph ^= 1;
                }
                asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
            }
            return;
        }
    }
    if (warp == NCW) {
        // ------------------------------------------------ TMA producer warp
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mapA));
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mapB));
            if constexpr (XS) asm volatile("prefetch.tensormap [%0];\n" ::"l"(&mapX));
            int stage = 0;
            unsigned phase = 0;
            unsigned xphase = 0;
            for (int64_t w = blockIdx.x; w < P.total_tiles; w += gridDim.x) {
                int64_t b, sp, mt, nt;
                ws_tile(P, w, b, sp, mt, nt);
                const int64_t kb = sp * P.kchunk, ke = min(P.K, kb + P.kchunk);
                if constexpr (EPI == EPI_RESID) {
                    // reference block of this tile -> Xs (after the previous
                    // tile's epilogue released it); lands during the k-loop
                    mbar_wait(xempty, xphase ^ 1);
                    mbar_expect_tx(xfull, (unsigned)(BM * BN * 8));
                    asm volatile(
                        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
                        "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(Xs)),
                        "l"(&mapX), "r"((int)(mt * BM)), "r"((int)(nt * BN)), "r"((int)b),
                        "r"((unsigned)__cvta_generic_to_shared(xfull))
                        : "memory");
                    xphase ^= 1;
                }
                for (int64_t k0 = kb; k0 < ke; k0 += BK) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], STAGE_BYTES);
                    double* as = As + stage * BM * BK;
                    double* bs = Bs + stage * BK * BN;
                    if constexpr (!AK)
                        tma_load_5d(as, &mapA, &full[stage], 0, (int)k0, (int)(mt * BM / 4), 0, (int)b);
                    else {
                        const int ks = P.a_kblock;
                        const int64_t kk = ks ? (k0 & ((1LL << ks) - 1)) : k0;
                        const int64_t kq = ks ? (k0 >> ks) : 0;
                        tma_load_5d(as, &mapA, &full[stage], 0, (int)(mt * BM), (int)(kk / 4), (int)kq, (int)b);
                    }
                    if constexpr (BNM)
                        tma_load_5d(bs, &mapB, &full[stage], 0, (int)k0, (int)(nt * BN / 4), 0, (int)b);
                    else {
                        const int ks = P.b_kblock;
                        const int64_t kk = ks ? (k0 & ((1LL << ks) - 1)) : k0;
                        const int64_t kq = ks ? (k0 >> ks) : 0;
                        tma_load_5d(bs, &mapB, &full[stage], 0, (int)(nt * BN), (int)(kk / 4), (int)kq, (int)b);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        return;
    }

    // ------------------------------------------------------ consumer warps
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp % WARPS_M, wn = warp / WARPS_M;
    int stage = 0;
    unsigned phase = 0;
    unsigned xph = 0;
    double sd = 0.0, sx = 0.0;  // RESID running sums (fixed tile order per CTA)

    for (int64_t w = blockIdx.x; w < P.total_tiles; w += gridDim.x) {
        int64_t b, sp, mt, nt;
        ws_tile(P, w, b, sp, mt, nt);
        const int64_t kb = sp * P.kchunk, ke = min(P.K, kb + P.kchunk);
        double acc[TM][TN][2];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

        for (int64_t k0 = kb; k0 < ke; k0 += BK) {
            mbar_wait(&full[stage], phase);
            const double* as = As + stage * BM * BK;
            const double* bs = Bs + stage * BK * BN;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double af[TM], bf[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i) {
                    const int m = wm * WM + i * 8 + g, k = kk + t;
                    af[i] = AK ? as[((k >> 2) * BM + m) * 4 + (k & 3)] : as[((m >> 2) * BK + k) * 4 + (m & 3)];
                }
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                    const int n = wn * WN + j * 8 + g, k = kk + t;
                    bf[j] = BNM ? bs[((n >> 2) * BK + k) * 4 + (n & 3)] : bs[((k >> 2) * BN + n) * 4 + (k & 3)];
                }
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) dmma884(acc[i][j], af[i], bf[j]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }

        const int64_t m0 = mt * BM, n0 = nt * BN;
        if constexpr (EPI == EPI_TSTORE) {
            // the store warp has read the previous tile out of Xs
            mbar_wait(xempty, xph ^ 1);
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int ml = wm * WM + i * 8 + g;
                        const int nl = wn * WN + j * 8 + 2 * t + e;
                        Xs[nl * BM + ml] = P.alpha * acc[i][j][e];  // rows / columns past M, N: not stored by TMA
                    }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> async proxy
            __syncwarp();
            if (lane == 0) mbar_arrive(xfull);
            xph ^= 1;
        } else if constexpr (EPI == EPI_STORE) {
            double* C = P.C + b * P.strideC + sp * P.strideCsplit;
            const double* Cin = P.Cin ? P.Cin + b * P.strideCin : nullptr;
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
        } else {
            mbar_wait(xfull, xph);
            xph ^= 1;
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int ml = wm * WM + i * 8 + g;
                        const int nl = wn * WN + j * 8 + 2 * t + e;
                        if (m0 + ml < P.M && n0 + nl < P.N) {
                            const double x = Xs[nl * BM + ml];
                            const double d = x - P.alpha * acc[i][j][e];
                            sd = fma(d, d, sd);
                            sx = fma(x, x, sx);
                        }
                    }
            __syncwarp();
            if (lane == 0) mbar_arrive(xempty);
        }
    }

    if constexpr (EPI == EPI_RESID) {
        // fixed-order CTA reduction over the consumer warps
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            sd += __shfl_xor_sync(0xffffffffu, sd, off);
            sx += __shfl_xor_sync(0xffffffffu, sx, off);
        }
        __shared__ double red[2 * 32];
        if (lane == 0) {
            red[2 * warp] = sd;
            red[2 * warp + 1] = sx;
        }
        asm volatile("bar.sync 1, %0;\n" ::"r"(NCW * 32));  // consumers only
        if (threadIdx.x == 0) {
            double a = 0.0, c = 0.0;
            for (int i = 0; i < NCW; ++i) {
                a += red[2 * i];
                c += red[2 * i + 1];
            }
            P.partial[2 * blockIdx.x] = a;
            P.partial[2 * blockIdx.x + 1] = c;
        }
    }
}

}  // namespace ppc
