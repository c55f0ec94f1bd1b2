// Host side of the warp-specialized TMA GEMM (dmma_gemm_ws.cuh): eligibility,
// tensor-map encoding (driver entry point, no -lcuda link), launch.
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdlib>
#include <mutex>

#include "dmma_gemm_ws.cuh"
#include "internal.h"

namespace ppc {

static std::atomic<int> g_gemm_path{-1};
int gemm_path() {
    int v = g_gemm_path.load();
    if (v < 0) {
        v = std::getenv("PPC_DISABLE_WS") ? 1 : 0;
        g_gemm_path.store(v);
    }
    return v;
}

namespace {

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

// 5-D map of an operand in the interleaved-quad smem layout.
//   mn_major: element (c, o) at base + c + o*ld (c = M/N index, o = k)
//   k-major:  element (o, c) at base + c + o*ld with c = k (contiguous), o = M/N,
//             optionally k-blocked: block kq at kq*kbstride.
bool make_map(CUtensorMap* map, const double* base, bool contiguous_is_k, int64_t cext, int64_t oext,
              int64_t ld, int64_t batch, int64_t bstride, int box_c, int box_o, int kshift, int64_t kbstride) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[5];
    cuuint64_t strides[4];
    cuuint32_t box[5];
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    if (!contiguous_is_k) {
        // d0 = c%4, d1 = o (k), d2 = c/4, d3 = 1, d4 = batch
        dims[0] = 4; dims[1] = (cuuint64_t)oext; dims[2] = (cuuint64_t)(cext / 4); dims[3] = 1;
        dims[4] = (cuuint64_t)batch;
        strides[0] = (cuuint64_t)ld * 8; strides[1] = 32; strides[2] = 32 * (cuuint64_t)(cext / 4);
        strides[3] = (cuuint64_t)bstride * 8;
        box[0] = 4; box[1] = (cuuint32_t)box_o; box[2] = (cuuint32_t)(box_c / 4); box[3] = 1; box[4] = 1;
    } else {
        // d0 = k%4, d1 = o (m/n), d2 = (k within block)/4, d3 = k block, d4 = batch
        const int64_t kb = kshift ? (1LL << kshift) : cext;
        const int64_t nb = kshift ? (cext + kb - 1) / kb : 1;
        dims[0] = 4; dims[1] = (cuuint64_t)oext; dims[2] = (cuuint64_t)(kb / 4); dims[3] = (cuuint64_t)nb;
        dims[4] = (cuuint64_t)batch;
        strides[0] = (cuuint64_t)ld * 8; strides[1] = 32;
        strides[2] = (cuuint64_t)(kshift ? kbstride : kb) * 8;
        strides[3] = (cuuint64_t)bstride * 8;
        box[0] = 4; box[1] = (cuuint32_t)box_o; box[2] = (cuuint32_t)(box_c / 4); box[3] = 1; box[4] = 1;
    }
    for (int i = 0; i < 4; ++i)
        if (strides[i] % 16 || strides[i] >= (1ULL << 40)) return false;
    if (strides[3] == 0) strides[3] = 16;  // batch 1: any legal stride
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES>
struct WsCfg {
    static constexpr int bm = BM, bn = BN;
    static constexpr size_t smem = (size_t)STAGES * (BM * 16 + 16 * BN) * 8 + 2 * STAGES * 8 + 128;
    template <bool AK, bool BNM, int EPI>
    static void launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& x, const WsParams& P,
                       int grid, cudaStream_t s) {
        auto k = dmma_gemm_ws_kernel<BM, BN, 16, WARPS_M, WARPS_N, STAGES, AK, BNM, EPI>;
        const size_t sm = smem + (EPI != EPI_STORE ? (size_t)BM * BN * 8 + 16 : 0);
        static std::atomic<uint64_t> set{0};
        once_per_device(set, [&] {
            PPC_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        });
        k<<<grid, ws_threads<BM, BN, WARPS_M, WARPS_N, EPI>(), sm, s>>>(a, b, x, P);
    }
};
using WsL = WsCfg<128, 128, 2, 4, 5>;
using WsR = WsCfg<128, 128, 2, 4, 3>;  // fused residual: 3 stages + the 128 KB X tile
using WsM = WsCfg<128, 64, 4, 2, 6>;
using WsT = WsCfg<128, 32, 4, 1, 8>;

template <class Cfg>
void dispatch(bool ak, bool bnm, int epi, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& x,
              const WsParams& P, int grid, cudaStream_t s) {
    if (!ak && !bnm && epi == EPI_STORE) return Cfg::template launch<false, false, EPI_STORE>(a, b, x, P, grid, s);
    if (!ak && bnm && epi == EPI_STORE) return Cfg::template launch<false, true, EPI_STORE>(a, b, x, P, grid, s);
    if (ak && !bnm && epi == EPI_STORE) return Cfg::template launch<true, false, EPI_STORE>(a, b, x, P, grid, s);
    fail(PPC_ARGUMENT, "gemm_ws: unsupported variant");
}

// the TMA-store epilogue (configurations whose operand ring leaves room for the output tile)
template <class Cfg>
void dispatch_tstore(bool ak, bool bnm, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                     const WsParams& P, int grid, cudaStream_t s) {
    if (!ak && !bnm) return Cfg::template launch<false, false, EPI_TSTORE>(a, b, c, P, grid, s);
    if (!ak && bnm) return Cfg::template launch<false, true, EPI_TSTORE>(a, b, c, P, grid, s);
    if (ak && !bnm) return Cfg::template launch<true, false, EPI_TSTORE>(a, b, c, P, grid, s);
    fail(PPC_ARGUMENT, "gemm_ws: unsupported variant");
}

// 3-D map of the residual reference X (M x N column-major, ld, batch stride):
// box = one BM x BN tile, written to smem as [n][m].
bool make_map_x(CUtensorMap* map, const double* X, int64_t M, int64_t N, int64_t ld, int64_t batch,
                int64_t bstride, int bm, int bn) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)M, (cuuint64_t)N, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)(bstride ? bstride : ld * N) * 8};
    cuuint32_t box[3] = {(cuuint32_t)bm, (cuuint32_t)bn, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (strides[0] % 16 || strides[1] % 16) return false;
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(X), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t short_k_cfg() {
    static const int64_t v = std::getenv("PPC_WS_SHORT_K") ? std::atoll(std::getenv("PPC_WS_SHORT_K")) : 256;
    return v;
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

// Returns false (nothing launched) when the problem does not fit the TMA path.
bool gemm_ws(const GemmDesc& d, int epi, const double* X, int64_t ldx, int64_t strideX, double* partials,
             int64_t* ctas_out, cudaStream_t s) {
    HostProf hp_("gemm_ws");
    if (gemm_path() == 1) return false;  // forced classic cp.async kernel
    if (d.M < 1 || d.N < 1 || d.K < 1) return false;
    if (d.zmap && d.zmap_extent < 1) return false;
    const int64_t map_batch = d.zmap ? d.zmap_extent : d.batch;
    if (d.a_kmajor && d.b_nmajor) return false;
    if (epi == EPI_RESID && (d.a_kmajor || !d.b_nmajor)) return false;
    // configuration
    int cfg;  // 0 = L, 1 = M, 2 = T
    if (d.symmetric) {
        cfg = 0;
    } else if (d.N <= 32) {
        cfg = 2;
    } else if (d.N <= 64) {
        cfg = 1;
    } else if (epi == EPI_STORE && d.K <= short_k_cfg()) {
        // short-K stores: the 128 x 128 consumers (64 accumulators a thread;
        // 168 registers with 9 warps, one SMSP holding 3 -> spills) ran at
        // 55% of the DMMA pipe; the 128 x 64 tile keeps everything in
        // registers (cfg4 inverse transform 1.71 -> 1.47 ms)
        cfg = 1;
    } else {
        cfg = 0;
    }
    const int bm = 128, bn = cfg == 0 ? 128 : (cfg == 1 ? 64 : 32), bk = 16;
    // big enough to be worth a persistent launch
    const int64_t mt = (d.M + bm - 1) / bm, nt = (d.N + bn - 1) / bn;
    const int64_t tiles = d.symmetric ? nt * (nt + 1) / 2 : mt * nt;
    if (d.symmetric && bm != bn) return false;
    const int64_t kchunk = d.kchunk > 0 ? d.kchunk : (d.splits > 1 ? ((d.K + d.splits - 1) / d.splits + 15) / 16 * 16 : d.K);
    if (d.splits > 1 && kchunk % bk) return false;
    const int64_t total = tiles * d.splits * d.batch;
    const double work = (double)d.M * d.N * d.K * d.batch;
    if (work < 5e8 || total < 16) return false;
    // alignment / extents for the 5-D maps
    if (!al16(d.A) || !al16(d.B) || (d.lda & 1) || (d.ldb & 1) || (d.strideA & 1) || (d.strideB & 1)) return false;
    if (d.a_kmajor ? (d.K % 4 && !d.kshift) : (d.M % 4)) return false;
    if (d.b_nmajor ? (d.N % 4) : (d.K % 4 && !d.kshift)) return false;
    if (d.kshift && ((1LL << d.kshift) % bk)) return false;
    CUtensorMap ma, mb, mx_;
    bool ok;
    if (!d.a_kmajor)
        ok = make_map(&ma, d.A, false, d.M, d.K, d.lda, map_batch, d.strideA, bm, bk, 0, 0);
    else
        ok = make_map(&ma, d.A, true, d.K, d.M, d.lda, map_batch, d.strideA, bk, bm, d.kshift, d.kbstride);
    if (!ok) return false;
    if (d.b_nmajor)
        ok = make_map(&mb, d.B, false, d.N, d.K, d.ldb, map_batch, d.strideB, bn, bk, 0, 0);
    else
        ok = make_map(&mb, d.B, true, d.K, d.N, d.ldb, map_batch, d.strideB, bk, bn, d.kshift, d.kbstride);
    if (!ok) return false;

    WsParams P{};
    P.M = d.M; P.N = d.N; P.K = d.K; P.batch = d.batch;
    P.mtiles = mt; P.ntiles = nt; P.tiles_per_batch = tiles; P.total_tiles = total;
    P.tri = d.symmetric ? 1 : 0;
    P.nfast = (mt > 1 && nt > 1) ? 1 : 0;
    P.kchunk = kchunk; P.splits = d.splits; P.strideCsplit = d.strideCsplit;
    P.C = d.C; P.ldc = d.ldc; P.strideC = d.strideC;
    P.Cin = d.Cin; P.ldcin = d.ldcin; P.strideCin = d.strideCin;
    P.alpha = d.alpha; P.beta = d.beta;
    P.X = X; P.ldx = ldx; P.strideX = strideX; P.partial = partials;
    P.zmap = d.zmap;
    P.a_kblock = d.a_kmajor ? d.kshift : 0;
    P.b_kblock = !d.b_nmajor ? d.kshift : 0;
    const int sms = ctx().sms;
    const int grid = (int)std::min<int64_t>(total, sms);
    if (epi == EPI_RESID) {
        // the fused residual stages X through shared memory: 128 x 128 tiles
        if (cfg != 0 || d.zmap || !X || (ldx & 1) || (strideX & 1) || !al16(X)) return false;
        if (!make_map_x(&mx_, X, d.M, d.N, ldx, d.batch, strideX, bm, bn)) return false;
    }
    if (ctas_out) *ctas_out = grid;
    if (!partials && epi == EPI_RESID) return true;  // sizing query only
    // plain stores of the 128 x 64 / 128 x 32 tiles drain through shared
    // memory and a TMA store (the map clips rows / columns past M, N)
    static const bool no_tstore = std::getenv("PPC_WS_NO_TSTORE") != nullptr;
    const bool tstore = !no_tstore && epi == EPI_STORE && cfg != 0 && !d.symmetric && d.splits == 1 &&
                        !(d.Cin && d.beta != 0.0) && al16(d.C) && !(d.ldc & 1) && !(d.strideC & 1) &&
                        make_map_x(&mx_, d.C, d.M, d.N, d.ldc, map_batch, d.strideC, bm, bn);
    if (epi == EPI_RESID) {
        WsR::launch<false, true, EPI_RESID>(ma, mb, mx_, P, grid, s);
    } else if (tstore) {
        if (cfg == 1)
            dispatch_tstore<WsM>(d.a_kmajor, d.b_nmajor, ma, mb, mx_, P, grid, s);
        else
            dispatch_tstore<WsT>(d.a_kmajor, d.b_nmajor, ma, mb, mx_, P, grid, s);
    } else {
        switch (cfg) {
            case 0: dispatch<WsL>(d.a_kmajor, d.b_nmajor, epi, ma, mb, ma, P, grid, s); break;
            case 1: dispatch<WsM>(d.a_kmajor, d.b_nmajor, epi, ma, mb, ma, P, grid, s); break;
            default: dispatch<WsT>(d.a_kmajor, d.b_nmajor, epi, ma, mb, ma, P, grid, s); break;
        }
    }
    count_launch();
    check_launch("dmma_gemm_ws");
    return true;
}

}  // namespace ppc

extern "C" int ppc_set_gemm_path(int mode) {
    if (mode < 0 || mode > 1) return PPC_ARGUMENT;
    ppc::g_gemm_path.store(mode);
    return 0;
}
