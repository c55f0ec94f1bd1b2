// Instantiation helpers for dmma_gemm_kernel: one translation unit per tile
// configuration (gemm_cfg_*.cu) so the 8 operand/epilogue variants of each
// configuration compile in parallel.
#pragma once

#include "dmma_gemm.cuh"
#include "internal.h"

namespace ppc {

template <int BM_, int BN_, int WARPS_M_, int WARPS_N_, int STAGES_>
struct TileCfg {
    static constexpr int BM = BM_, BN = BN_, BK = 16, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_,
                         STAGES = STAGES_;
    static constexpr int threads = WARPS_M * WARPS_N * 32;
    static constexpr size_t smem = (size_t)STAGES * (BM * BK + BK * BN) * sizeof(double);
};

template <class Cfg, bool AK, bool BNM, int VEC, int EPI>
void launch_variant(const GemmParams& P, dim3 grid, cudaStream_t s) {
    auto kern = dmma_gemm_kernel<Cfg::BM, Cfg::BN, Cfg::BK, Cfg::WARPS_M, Cfg::WARPS_N,
                                 Cfg::STAGES, AK, BNM, VEC, EPI>;
    static std::atomic<uint64_t> attr_set{0};  // per instantiation, per device
    once_per_device(attr_set, [&] {
        PPC_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)Cfg::smem));
    });
    kern<<<grid, Cfg::threads, Cfg::smem, s>>>(P);
}

// Dispatch over the supported operand orientations. (A K-major, B N-major)
// is never needed by the engine and is rejected.
template <class Cfg>
void launch_cfg(const GemmParams& P, dim3 grid, bool ak, bool bnm, bool vec2, int epi,
                cudaStream_t s) {
#define PPC_V(AKV, BNV, VV, EV) \
    if (ak == AKV && bnm == BNV && (vec2 ? 2 : 1) == VV && epi == EV) \
        return launch_variant<Cfg, AKV, BNV, VV, EV>(P, grid, s);
    PPC_V(false, false, 2, EPI_STORE)
    PPC_V(false, false, 1, EPI_STORE)
    PPC_V(false, true, 2, EPI_STORE)
    PPC_V(false, true, 1, EPI_STORE)
    PPC_V(true, false, 2, EPI_STORE)
    PPC_V(true, false, 1, EPI_STORE)
    PPC_V(false, true, 2, EPI_RESID)
    PPC_V(false, true, 1, EPI_RESID)
#undef PPC_V
    fail(PPC_ARGUMENT, "gemm: unsupported operand orientation / epilogue combination");
}

// Tile configurations (BM, BN, warps_m, warps_n, stages).
using CfgL = TileCfg<128, 128, 2, 4, 4>;    // square, compute-bound
using CfgM = TileCfg<128, 64, 4, 2, 4>;
using CfgS = TileCfg<64, 64, 2, 2, 3>;      // small problems: more CTAs
using CfgT32 = TileCfg<128, 32, 4, 1, 4>;   // tall-skinny forward transforms
using CfgT24 = TileCfg<128, 24, 4, 1, 4>;
using CfgT16 = TileCfg<128, 16, 4, 1, 4>;
using CfgT8 = TileCfg<128, 8, 4, 1, 4>;

#define PPC_DECLARE_CFG(Cfg)                                                               \
    extern template void launch_cfg<Cfg>(const GemmParams&, dim3, bool, bool, bool, int, \
                                         cudaStream_t);
PPC_DECLARE_CFG(CfgL)
PPC_DECLARE_CFG(CfgM)
PPC_DECLARE_CFG(CfgS)
PPC_DECLARE_CFG(CfgT32)
PPC_DECLARE_CFG(CfgT24)
PPC_DECLARE_CFG(CfgT16)
PPC_DECLARE_CFG(CfgT8)
#undef PPC_DECLARE_CFG

}  // namespace ppc
