// Host-side dispatch of the FP64 DMMA GEMM: tile-configuration choice,
// vector-width eligibility and grid construction.
#include "gemm_impl.cuh"

namespace ppc {

namespace {

enum CfgId { L, M, S, T32, T24, T16, T8 };

struct CfgInfo {
    int bm, bn;
};
constexpr CfgInfo kInfo[] = {{128, 128}, {128, 64}, {64, 64}, {128, 32},
                             {128, 24},  {128, 16}, {128, 8}};

CfgId choose(const GemmDesc& d) {
    const int64_t work_ctas_L = ((d.M + 127) / 128) * ((d.N + 127) / 128) * d.batch * d.splits;
    if (d.N <= 8) return T8;
    if (d.N <= 16) return T16;
    if (d.N <= 24) return T24;
    if (d.N <= 32) return T32;
    if (d.symmetric) return work_ctas_L >= 296 ? L : S;
    // M <= 64: the 128-row tile would spend half its MMAs on padding rows
    if (d.N <= 64) return (d.M > 64 && ((d.M + 127) / 128) * d.batch * d.splits >= 148) ? M : S;
    return work_ctas_L >= 148 ? L : S;
}

bool even(int64_t v) { return (v & 1) == 0; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// 16-byte cp.async needs every contiguous-dimension extent, leading
// dimension, batch stride and split boundary to be even, and 16 B bases.
bool vec2_ok(const GemmDesc& d, int64_t kchunk) {
    const int64_t a_c = d.a_kmajor ? d.K : d.M;
    const int64_t b_c = d.b_nmajor ? d.N : d.K;
    return even(a_c) && even(b_c) && even(d.lda) && even(d.ldb) && even(d.strideA) &&
           even(d.strideB) && even(kchunk) && aligned16(d.A) && aligned16(d.B);
}

void fill(GemmParams& P, const GemmDesc& d, int64_t kchunk) {
    P = GemmParams{};
    P.M = d.M; P.N = d.N; P.K = d.K;
    P.A = d.A; P.lda = d.lda; P.strideA = d.strideA;
    P.B = d.B; P.ldb = d.ldb; P.strideB = d.strideB;
    P.C = d.C; P.ldc = d.ldc; P.strideC = d.strideC;
    P.Cin = d.Cin; P.ldcin = d.ldcin; P.strideCin = d.strideCin;
    P.alpha = d.alpha; P.beta = d.beta;
    P.kchunk = kchunk;
    P.strideCsplit = d.strideCsplit;
    P.tri = d.symmetric ? 1 : 0;
    P.kshift = d.kshift;
    P.kbstride = d.kbstride;
    P.zmap = d.zmap;
}

void validate(const GemmDesc& d) {
    if (d.M < 0 || d.N < 0 || d.K < 0 || d.batch < 1 || d.splits < 1)
        fail(PPC_ARGUMENT, "gemm: bad extents");
    if (d.a_kmajor && d.b_nmajor)
        fail(PPC_ARGUMENT, "gemm: (A^T, B^T) orientation not supported");
    if (d.symmetric && d.M != d.N) fail(PPC_ARGUMENT, "gemm: symmetric needs M == N");
    if (d.batch > 65535 || d.splits > 65535) fail(PPC_ARGUMENT, "gemm: batch/splits too large");
    if (d.kshift && (d.b_nmajor || !d.a_kmajor))
        fail(PPC_ARGUMENT, "gemm: k-blocked addressing needs K-major A and B");
}

void launch(CfgId id, const GemmParams& P, dim3 grid, const GemmDesc& d, bool v2, int epi,
            cudaStream_t s) {
    switch (id) {
        case L: launch_cfg<CfgL>(P, grid, d.a_kmajor, d.b_nmajor, v2, epi, s); break;
        case M: launch_cfg<CfgM>(P, grid, d.a_kmajor, d.b_nmajor, v2, epi, s); break;
        case S: launch_cfg<CfgS>(P, grid, d.a_kmajor, d.b_nmajor, v2, epi, s); break;
        case T32: launch_cfg<CfgT32>(P, grid, d.a_kmajor, d.b_nmajor, v2, epi, s); break;
        case T24: launch_cfg<CfgT24>(P, grid, d.a_kmajor, d.b_nmajor, v2, epi, s); break;
        case T16: launch_cfg<CfgT16>(P, grid, d.a_kmajor, d.b_nmajor, v2, epi, s); break;
        case T8: launch_cfg<CfgT8>(P, grid, d.a_kmajor, d.b_nmajor, v2, epi, s); break;
    }
    count_launch();
    check_launch("dmma_gemm");
}

dim3 grid_for(CfgId id, const GemmDesc& d, int64_t* ctas) {
    const CfgInfo ci = kInfo[id];
    const int64_t mt = (d.M + ci.bm - 1) / ci.bm, nt = (d.N + ci.bn - 1) / ci.bn;
    int64_t tiles = d.symmetric ? nt * (nt + 1) / 2 : mt * nt;
    if (tiles > 0x7fffffffLL) fail(PPC_ARGUMENT, "gemm: too many tiles");
    if (ctas) *ctas = tiles * d.splits * d.batch;
    return dim3((unsigned)tiles, (unsigned)d.splits, (unsigned)d.batch);
}

int64_t kchunk_of(const GemmDesc& d) {
    if (d.kchunk > 0) return d.kchunk;
    if (d.splits <= 1) return d.K > 0 ? d.K : 1;
    int64_t kc = (d.K + d.splits - 1) / d.splits;
    kc = (kc + 15) / 16 * 16;  // split boundaries on BK multiples
    return kc;
}

}  // namespace

void gemm(const GemmDesc& d, cudaStream_t s) {
    HostProf hp_("gemm");
    validate(d);
    if (d.M == 0 || d.N == 0) return;
    if (d.allow_ws && gemm_ws(d, EPI_STORE, nullptr, 0, 0, nullptr, nullptr, s)) return;
    const CfgId id = choose(d);
    const int64_t kchunk = kchunk_of(d);
    GemmParams P;
    fill(P, d, kchunk);
    // m-fast raster keeps consecutive CTAs on one B panel when there are few
    // n tiles (tall-skinny); n-fast keeps them on one A panel otherwise.
    P.nfast = ((d.M + kInfo[id].bm - 1) / kInfo[id].bm) > 1 &&
                      ((d.N + kInfo[id].bn - 1) / kInfo[id].bn) > 1
                  ? 1
                  : 0;
    const dim3 grid = grid_for(id, d, nullptr);
    launch(id, P, grid, d, vec2_ok(d, kchunk), EPI_STORE, s);
}

int64_t gemm_residual_ctas(const GemmDesc& d, const double* X, int64_t ldx, int64_t strideX) {
    int64_t ctas = 0;
    if (d.allow_ws && gemm_ws(d, EPI_RESID, X, ldx, strideX, nullptr, &ctas, nullptr)) return ctas;
    grid_for(choose(d), d, &ctas);
    return ctas;
}

void gemm_residual(const GemmDesc& d, const double* X, int64_t ldx, int64_t strideX,
                   double* partials, cudaStream_t s) {
    validate(d);
    if (d.symmetric || d.splits != 1) fail(PPC_ARGUMENT, "gemm_residual: plain tiling only");
    if (d.M == 0 || d.N == 0) return;
    if (d.allow_ws && gemm_ws(d, EPI_RESID, X, ldx, strideX, partials, nullptr, s)) return;
    const CfgId id = choose(d);
    const int64_t kchunk = kchunk_of(d);
    GemmParams P;
    fill(P, d, kchunk);
    P.nfast = 1;
    P.X = X;
    P.ldx = ldx;
    P.strideX = strideX;
    P.partial = partials;
    const dim3 grid = grid_for(id, d, nullptr);
    launch(id, P, grid, d, vec2_ok(d, kchunk), EPI_RESID, s);
}

}  // namespace ppc
