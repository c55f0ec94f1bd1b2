// Device-level hot path (see engine.h). Every GEMM-shaped stage runs on the
// FP64 DMMA kernel (dmma_gemm.cuh); reductions are fixed-order.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "dmma_gemm.cuh"
#include "engine.h"
#include "internal.h"
#include "jacobi.cuh"
#include "kernels.cuh"
#include "ozaki.h"
#include "slice_svd.cuh"

namespace ppc {

void mode3(const double* T, int64_t N, int64_t n3, const double* M, int64_t q, bool trans_m,
           double* out, double alpha, cudaStream_t s) {
    StageTimer tm(trans_m ? "mode3_fwd" : "mode3_inv", s, 2.0 * N * n3 * q,
                  8.0 * (N * n3 + N * q + n3 * q));
    GemmDesc d;
    d.M = N; d.N = q; d.K = n3;
    d.A = T; d.lda = N; d.a_kmajor = false;
    d.B = M;
    if (trans_m) {  // B(k,n) = M[k + n*n3]
        d.ldb = n3; d.b_nmajor = false;
    } else {        // B(k,n) = M^T(k,n) = M[n + k*q]
        d.ldb = q; d.b_nmajor = true;
    }
    d.C = out; d.ldc = N;
    d.alpha = alpha;
    gemm(d, s);
}

void facewise(const double* A, int64_t n1, int64_t m, int64_t p, const double* B, int64_t n2,
              double* C, cudaStream_t s) {
    StageTimer tm("facewise", s, 2.0 * n1 * m * n2 * p, 8.0 * p * (n1 * m + m * n2 + n1 * n2));
    GemmDesc d;
    d.M = n1; d.N = n2; d.K = m; d.batch = p;
    d.A = A; d.lda = n1; d.strideA = n1 * m;
    d.B = B; d.ldb = m; d.strideB = m * n2;
    d.C = C; d.ldc = n1; d.strideC = n1 * n2;
    gemm(d, s);
}

namespace {

// The transform-domain facewise product on the INT8 tensor cores (Ozaki):
// Ch_i = Ah_i Bh_i with Ah_i^T (slice-wise transpose, K = m contiguous) and
// Bh_i split into digits along m; Bd may carry B's digits from a previous
// call (host pipeline: one B for every A row block). Rows run in blocks of
// kFaceRows: a block whose rows (or B's columns) fail the dynamic-range gate
// (ozaki_peak_ratios) is computed on FP64 DMMA instead, so the host pipeline
// (one call per row block) and the device call decide every row the same way
// and stay bitwise equal. Returns false when nothing ran on the INT8 path
// (the caller then runs the DMMA facewise on all rows).
constexpr int64_t kFaceRows = 128;

void facewise_rows(const double* Ah, int64_t n1, int64_t i0, int64_t bi, int64_t m, int64_t p, const double* Bh,
                   int64_t n2, double* Ch, int64_t ldc, int64_t strideC, cudaStream_t s) {
    GemmDesc d;  // rows [i0, i0 + bi) of every slice
    d.M = bi; d.N = n2; d.K = m; d.batch = p;
    d.A = Ah + i0; d.lda = n1; d.strideA = n1 * m;
    d.B = Bh; d.ldb = m; d.strideB = m * n2;
    d.C = Ch + i0; d.ldc = ldc; d.strideC = strideC;
    gemm(d, s);
}

// Ch (slice i at Ch + i*strideC, leading dimension ldc; n1 x n2 per slice).
bool facewise_ozaki(const double* Ah, int64_t n1, int64_t m, int64_t p, const double* Bh, int64_t n2, double* Ch,
                    OzakiDigits& Bd, bool& b_ready, double& b_peak, cudaStream_t s, int64_t ldc = 0,
                    int64_t strideC = 0) {
    if (ldc <= 0) ldc = n1;
    if (strideC <= 0) strideC = n1 * n2;
    if (!ozaki_gemm_eligible(n1, m) || n2 < 64) return false;
    if (b_ready && b_peak > kOzakiPeakGate) return false;
    StageTimer tm("facewise", s, 2.0 * n1 * m * n2 * p, 8.0 * p * (n1 * m + m * n2 + n1 * n2));
    // both operands split and their gate values computed on the device, then
    // one host read for the decision (B's only with the first row block)
    // A-hat's slices split as their transposes (m x n1, K-major), read in place
    OzakiDigits Ad;
    Ad.split(Ah, n1, n1 * m, m, n1, m, p, s, nullptr, 0, 0, 0, nullptr, 6, 0, 0, nullptr, 0, true);
    const int64_t ng = ozaki_peak_groups(Ad, kFaceRows);
    DeviceBuffer peaks(sizeof(double) * (ng + 1));
    ozaki_peak_ratios_async(Ad, m, kFaceRows, peaks.d(), s);
    if (!b_ready) {
        Bd.split(Bh, m, m * n2, m, n2, m, p, s);
        ozaki_peak_ratios_async(Bd, m, n2, peaks.d() + ng, s);
    }
    std::vector<double> a_peak((size_t)ng + 1);
    // (not a cudaMemcpyAsync: in the host pipeline it would wait on the copy
    // engine for the previous block's C rows to finish their way down)
    read_small(peaks.d(), a_peak.data(), (size_t)(b_ready ? ng : ng + 1), s);
    if (!b_ready) {
        b_peak = a_peak[ng];
        b_ready = true;
    }
    a_peak.resize((size_t)ng);
    if (b_peak > kOzakiPeakGate) return false;
    // a short last block runs on DMMA too, as it does as its own host-pipeline call
    auto int8_rows = [&](size_t g) {
        return a_peak[g] <= kOzakiPeakGate && n1 - (int64_t)g * kFaceRows >= kFaceRows;
    };
    bool any = false;
    for (size_t g = 0; g < a_peak.size(); ++g) any |= int8_rows(g);
    if (!any) return false;
    ozaki_gemm(Ad, Bd, p, nullptr, Ch, ldc, strideC, s);
    for (size_t g = 0; g < a_peak.size(); ++g)
        if (!int8_rows(g)) {
            const int64_t i0 = (int64_t)g * kFaceRows;
            facewise_rows(Ah, n1, i0, std::min(kFaceRows, n1 - i0), m, p, Bh, n2, Ch, ldc, strideC, s);
        }
    return true;
}

}  // namespace

void facewise_auto(const double* Ah, int64_t n1, int64_t m, int64_t p, const double* Bh, int64_t n2, double* Ch,
                   int64_t ldc, int64_t strideC, cudaStream_t s) {
    OzakiDigits bd;
    bool b_ready = false;
    double b_peak = 0.0;
    if (!facewise_ozaki(Ah, n1, m, p, Bh, n2, Ch, bd, b_ready, b_peak, s, ldc, strideC)) {
        StageTimer tm("facewise", s, 2.0 * n1 * m * n2 * p, 8.0 * p * (n1 * m + m * n2 + n1 * n2));
        facewise_rows(Ah, n1, 0, n1, m, p, Bh, n2, Ch, ldc, strideC, s);
    }
}

namespace {

}  // namespace

void star_inverse(const double* Ch, int64_t N, int64_t p, const double* Q, int64_t n3, double scale, double* C,
                  cudaStream_t s) {
    if (!ozaki_star_inverse(Ch, N, p, Q, n3, scale, C, N, s)) mode3(Ch, N, p, Q, n3, false, C, scale, s);
}

void star_q(const double* A, int64_t n1, int64_t m, int64_t n3, const double* B, int64_t n2,
            const double* Q, int64_t p, double scale, double* C, cudaStream_t s) {
    DeviceBuffer ah(sizeof(double) * n1 * m * p), bh(sizeof(double) * m * n2 * p),
        ch(sizeof(double) * n1 * n2 * p);
    mode3(A, n1 * m, n3, Q, p, true, ah.d(), 1.0, s);   // A x3 Q^T
    mode3(B, m * n2, n3, Q, p, true, bh.d(), 1.0, s);   // B x3 Q^T
    OzakiDigits bd;
    bool b_ready = false;
    double b_peak = 0.0;
    if (!facewise_ozaki(ah.d(), n1, m, p, bh.d(), n2, ch.d(), bd, b_ready, b_peak, s))
        facewise(ah.d(), n1, m, p, bh.d(), n2, ch.d(), s);   // facewise
    star_inverse(ch.d(), n1 * n2, p, Q, n3, scale, C, s);  // x3 Q, scaled
}

namespace {

struct Event {
    cudaEvent_t e = nullptr;
    Event() { PPC_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
    ~Event() { cudaEventDestroy(e); }
    void record(cudaStream_t s) { PPC_CUDA_CHECK(cudaEventRecord(e, s)); }
    void wait_on(cudaStream_t s) { PPC_CUDA_CHECK(cudaStreamWaitEvent(s, e, 0)); }
};

}  // namespace

void star_q_host(const double* hA, int64_t n1, int64_t m, int64_t n3, const double* hB, int64_t n2,
                 const double* hQ, int64_t p, double scale, double* hC, cudaStream_t s) {
    // 2-D tiling: A in blocks of kFaceRows rows, B in blocks of kFaceRows
    // lateral columns. Tile (I, J) of C needs only A block I and B block J, so
    // the first rows of C start their way down after two blocks have come up,
    // not after all of B (the row-block pipeline before this: 70 ms at cfg4,
    // of which 22 before the first download).
    //  - every upload is enqueued at once on the H2D stream, alternating A and
    //    B blocks, each into its own device buffer;
    //  - a block is transformed, split into digits and gated as it lands;
    //  - each arrival enables the tiles it completes: facewise product, inverse
    //    transform, one 3-D copy down (D2H stream), four tile buffers rotating.
    // Same bits as star_q on device copies: the INT8 digits of a row / column,
    // the exact integer sums, the row-wise inverse transform and the DMMA
    // k-order do not depend on the tiling. B-hat's gate is one value over all
    // of B (as in star_q): tiles run on the INT8 path until a B block fails it;
    // then every tile so far is redone on FP64 DMMA, as star_q would have.
    cudaStream_t up = copy_stream(), down = copy_out_stream();
    // PPC_STARQ_TRACE: timed events on the three streams, printed at the end
    static const bool trace = std::getenv("PPC_STARQ_TRACE") != nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    auto mark = [&](const char* what, int64_t i, int64_t j, cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t e;
        PPC_CUDA_CHECK(cudaEventCreate(&e));
        PPC_CUDA_CHECK(cudaEventRecord(e, st));
        marks.emplace_back(std::string(what) + " " + std::to_string(i) + (j >= 0 ? "," + std::to_string(j) : ""), e);
    };
    mark("start", 0, -1, s);
    struct Block {
        int64_t o = 0, n = 0;         // first row / column, extent
        DeviceBuffer hat;             // A blocks: the transform (compact); B's go into bh
        OzakiDigits dig;
        double peak = 0.0;
        std::unique_ptr<Event> landed;
    };
    auto blocks_of = [](int64_t n, bool merge_short) {
        std::vector<Block> v;
        for (int64_t o = 0; o < n;) {
            int64_t len = std::min(kFaceRows, n - o);
            // lateral blocks: a short tail joins the last block (the INT8 product wants >= 64 columns)
            if (merge_short && n - o < kFaceRows + 64) len = n - o;
            v.emplace_back();
            v.back().o = o;
            v.back().n = len;
            o += len;
        }
        return v;
    };
    std::vector<Block> ab = blocks_of(n1, false), bb = blocks_of(n2, true);
    const int64_t nI = (int64_t)ab.size(), nJ = (int64_t)bb.size();
    const bool int8_ok = ozaki_gemm_eligible(n1, m) && n2 >= 64;  // star_q's shape test
    DeviceBuffer q(sizeof(double) * n3 * p);
    for (Block& x : ab) x.hat = DeviceBuffer(sizeof(double) * x.n * m * p);
    DeviceBuffer bh(sizeof(double) * m * n2 * p);  // B-hat whole: slice i at i * m * n2 (star_q's layout)
    // the blocks as uploaded: rings of kRing buffers per operand, so the uploads
    // run kRing - 1 steps ahead of the transforms whatever the tensors' size
    constexpr int kRing = 4;
    int64_t maxn = 0;
    for (const Block& x : bb) maxn = std::max(maxn, x.n);
    const int64_t BI = ab.empty() ? 0 : ab[0].n;
    DeviceBuffer araw[kRing], braw[kRing];
    Event a_done[kRing], b_done[kRing];  // the transform reading the slot is enqueued
    for (int r = 0; r < kRing; ++r) {
        araw[r] = DeviceBuffer(sizeof(double) * BI * m * n3);
        braw[r] = DeviceBuffer(sizeof(double) * m * maxn * n3);
    }
    Event ready;
    ready.record(s);  // buffers allocated on s
    ready.wait_on(up);
    PPC_CUDA_CHECK(cudaMemcpyAsync(q.d(), hQ, sizeof(double) * n3 * p, cudaMemcpyHostToDevice, up));
    // 1. uploads, alternating A and B blocks (step t: A block t, then B block t)
    const int64_t steps = std::max(nI, nJ);
    auto upload = [&](int64_t t) {
        if (t >= steps) return;
        const int r = (int)(t % kRing);
        if (t < nI) {
            Block& x = ab[(size_t)t];  // rows [o, o+n) of every lateral slice: n x (m n3), compact
            if (t >= kRing) a_done[r].wait_on(up);
            PPC_CUDA_CHECK(cudaMemcpy2DAsync(araw[r].d(), sizeof(double) * x.n, hA + x.o, sizeof(double) * n1,
                                             sizeof(double) * x.n, m * n3, cudaMemcpyHostToDevice, up));
            x.landed = std::make_unique<Event>();
            x.landed->record(up);
            mark("A block up", t, -1, up);
        }
        if (t < nJ) {
            Block& x = bb[(size_t)t];  // columns [o, o+n) of every frontal slice: (m n) x n3, compact
            if (t >= kRing) b_done[r].wait_on(up);
            PPC_CUDA_CHECK(cudaMemcpy2DAsync(braw[r].d(), sizeof(double) * m * x.n, hB + x.o * m,
                                             sizeof(double) * m * n2, sizeof(double) * m * x.n, n3,
                                             cudaMemcpyHostToDevice, up));
            x.landed = std::make_unique<Event>();
            x.landed->record(up);
            mark("B block up", t, -1, up);
        }
    };
    for (int64_t t = 0; t < kRing; ++t) upload(t);
    // 2. tiles
    constexpr int kBufs = 4;
    DeviceBuffer chb[kBufs], cb[kBufs];
    Event c_free[kBufs];
    for (int u = 0; u < kBufs; ++u) {
        chb[u] = DeviceBuffer(sizeof(double) * BI * maxn * p);
        cb[u] = DeviceBuffer(sizeof(double) * BI * maxn * n3);
        c_free[u].record(s);
    }
    bool b_bad = !int8_ok;  // B-hat failed the gate (or the shape never qualified): DMMA everywhere
    const bool inv_int8 = ((n1 * n2) & 1) == 0;
    int64_t ntile = 0;
    auto tile = [&](int64_t I, int64_t J, bool dmma) {
        Block& a = ab[(size_t)I];
        Block& b = bb[(size_t)J];
        const int u = (int)(ntile++ % kBufs);
        c_free[u].wait_on(s);  // this buffer's previous tile is down
        // the INT8 path as in facewise_ozaki: whole kFaceRows row blocks passing the gate
        const bool int8 = !dmma && a.n >= kFaceRows && a.peak <= kOzakiPeakGate;
        {
            StageTimer tm("facewise", s, 2.0 * a.n * m * b.n * p, 8.0 * p * (a.n * m + m * b.n + a.n * b.n));
            if (int8) {
                ozaki_gemm(a.dig, b.dig, p, nullptr, chb[u].d(), a.n, a.n * b.n, s);
            } else {
                GemmDesc d;
                d.M = a.n; d.N = b.n; d.K = m; d.batch = p;
                d.A = a.hat.d(); d.lda = a.n; d.strideA = a.n * m;
                d.B = bh.d() + b.o * m; d.ldb = m; d.strideB = m * n2;
                d.C = chb[u].d(); d.ldc = a.n; d.strideC = a.n * b.n;
                gemm(d, s);
            }
        }
        // x3 Q, scaled; on the path star_q takes for the whole product (its
        // INT8 kernel wants an even leading dimension: n1 n2 there, the tile's
        // row count here, which is even whenever n1 n2 is)
        if (!(inv_int8 && ozaki_star_inverse(chb[u].d(), a.n * b.n, p, q.d(), n3, scale, cb[u].d(), a.n * b.n, s)))
            mode3(chb[u].d(), a.n * b.n, p, q.d(), n3, false, cb[u].d(), scale, s);
        Event done;
        done.record(s);
        done.wait_on(down);
        mark("tile computed", I, J, s);
        cudaMemcpy3DParms cp{};
        cp.srcPtr = make_cudaPitchedPtr(cb[u].d(), sizeof(double) * a.n, sizeof(double) * a.n, (size_t)b.n);
        cp.dstPtr = make_cudaPitchedPtr(hC + a.o + b.o * n1, sizeof(double) * n1, sizeof(double) * n1, (size_t)n2);
        cp.extent = make_cudaExtent(sizeof(double) * a.n, (size_t)b.n, (size_t)n3);
        cp.kind = cudaMemcpyDeviceToHost;
        PPC_CUDA_CHECK(cudaMemcpy3DAsync(&cp, down));
        c_free[u].record(down);
        mark("tile down", I, J, down);
    };
    DeviceBuffer peaks(sizeof(double));
    // every tile among rows [0, ni) x columns [0, nj) again, on DMMA
    auto redo = [&](int64_t ni, int64_t nj) {
        for (int64_t I = 0; I < ni; ++I)
            for (int64_t J = 0; J < nj; ++J) tile(I, J, true);
    };
    for (int64_t t = 0; t < steps; ++t) {
        const int r = (int)(t % kRing);
        if (t > 0) upload(t - 1 + kRing);  // into the slots step t - 1's transforms have read
        if (t < nI) {  // A block t: transform, digits, gate; then its tiles against the B blocks so far
            Block& x = ab[(size_t)t];
            x.landed->wait_on(s);
            mode3(araw[r].d(), x.n * m, n3, q.d(), p, true, x.hat.d(), 1.0, s);  // A_blk x3 Q^T
            a_done[r].record(s);
            if (!b_bad && x.n >= kFaceRows) {
                x.dig.split(x.hat.d(), x.n, x.n * m, m, x.n, m, p, s, nullptr, 0, 0, 0, nullptr, 6, 0, 0, nullptr, 0,
                            true);
                ozaki_peak_ratios_async(x.dig, m, kFaceRows, peaks.d(), s);
                read_small(peaks.d(), &x.peak, 1, s);
            }
            for (int64_t J = 0; J < std::min(t, nJ); ++J) tile(t, J, b_bad);
        }
        if (t < nJ) {  // B block t: transform, digits, gate; then its tiles against the A blocks so far
            Block& x = bb[(size_t)t];
            x.landed->wait_on(s);
            {
                StageTimer tm("mode3_fwd", s, 2.0 * m * x.n * n3 * p, 8.0 * (m * x.n * (n3 + p) + n3 * p));
                GemmDesc d;  // B-hat rows [o m, (o + n) m) of every slice = those tubes x Q
                d.M = m * x.n; d.N = p; d.K = n3;
                d.A = braw[r].d(); d.lda = m * x.n;
                d.B = q.d(); d.ldb = n3;
                d.C = bh.d() + x.o * m; d.ldc = m * n2;
                gemm(d, s);
            }
            b_done[r].record(s);
            if (!b_bad) {
                x.dig.split(bh.d() + x.o * m, m, m * n2, m, x.n, m, p, s);
                ozaki_peak_ratios_async(x.dig, m, x.n, peaks.d(), s);
                read_small(peaks.d(), &x.peak, 1, s);
                if (x.peak > kOzakiPeakGate) {
                    // this B block fails the gate: star_q runs the whole product on DMMA
                    b_bad = true;
                    redo(std::min(t + 1, nI), t);
                }
            }
            for (int64_t I = 0; I < std::min(t + 1, nI); ++I) tile(I, t, b_bad);
        }
    }
    if (trace) {
        PPC_CUDA_CHECK(cudaStreamSynchronize(down));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
        for (size_t i = 1; i < marks.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[0].second, marks[i].second);
            std::fprintf(stderr, "[starq trace] %8.2f ms  %s\n", ms, marks[i].first.c_str());
        }
        for (auto& mk : marks) cudaEventDestroy(mk.second);
    }
    Event all_down;
    all_down.record(down);
    all_down.wait_on(s);  // the stream-ordered frees below come after the last D2H
}

void sumsq(const double* a, const double* b, int64_t count, double sums[2], cudaStream_t s) {
    DeviceBuffer part(sizeof(double) * 2 * (kReduceBlocks + 1));
    double* fin = part.d() + 2 * kReduceBlocks;
    launch_sumsq_partials(a, b, count, part.d(), s);
    launch_reduce_pairs(part.d(), kReduceBlocks, fin, s);
    PPC_CUDA_CHECK(cudaMemcpyAsync(sums, fin, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
}

namespace {
// Fused residual GEMM: {sum (X - alpha op(A)op(B))^2, sum X^2} as host doubles.
std::array<double, 2> residual_sums(const GemmDesc& d, const double* X, int64_t ldx,
                                    int64_t strideX, cudaStream_t s) {
    // a tall product with a short inner dimension (the residual through Q at
    // small p): streamed, one row per thread (kernels.cu smallk_residual)
    static const bool no_smallk = std::getenv("PPC_NO_SMALLK") != nullptr;
    const bool smallk = !no_smallk && d.batch == 1 && d.K >= 1 && d.K <= 32 && d.M >= 4096 && !d.a_kmajor &&
                        d.b_nmajor && d.alpha == 1.0;
    const int64_t ctas = smallk ? smallk_residual_ctas(d.M, d.N) : gemm_residual_ctas(d, X, ldx, strideX);
    DeviceBuffer part(sizeof(double) * 2 * (ctas + 1));
    if (smallk)
        launch_smallk_residual(d.A, d.lda, d.B, d.ldb, X, ldx, d.M, d.N, d.K, part.d(), s);
    else
        gemm_residual(d, X, ldx, strideX, part.d(), s);
    double* fin = part.d() + 2 * ctas;
    launch_reduce_pairs(part.d(), ctas, fin, s);
    std::array<double, 2> out{};
    PPC_CUDA_CHECK(cudaMemcpyAsync(out.data(), fin, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    return out;
}
}  // namespace

std::array<double, 2> projection_residual(const double* T, int64_t N, int64_t n3, const double* Q,
                                          int64_t p, const double* coeff, cudaStream_t s) {
    DeviceBuffer cbuf;
    if (!coeff) {
        cbuf = DeviceBuffer(sizeof(double) * N * p);
        mode3(T, N, n3, Q, p, true, cbuf.d(), 1.0, s);
        coeff = cbuf.d();
    }
    // residual of T against coeff (N x p) * Q^T (p x n3): B(k,n) = Q[n + k*n3]
    GemmDesc d;
    d.M = N; d.N = n3; d.K = p;
    d.A = coeff; d.lda = N;
    d.B = Q; d.ldb = n3; d.b_nmajor = true;
    return residual_sums(d, T, N, 0, s);
}

void require_finite(const double* x, int64_t n, const char* who, cudaStream_t s) {
    FiniteFlag nf(s);
    launch_nonfinite(x, n, nf.d(), s);
    nf.check(s, who);
}

void core_from_factors(const double* U, const double* S, const double* V, int64_t n1, int64_t n2,
                       int64_t p, int64_t k, double* Chat, cudaStream_t s, int64_t kstride) {
    if (kstride <= 0) kstride = k;
    if (k == 0) {  // an all-zero multirank: the core is zero
        PPC_CUDA_CHECK(cudaMemsetAsync(Chat, 0, sizeof(double) * n1 * n2 * p, s));
        return;
    }
    DeviceBuffer us(sizeof(double) * n1 * k * p);
    if (kstride == k)
        launch_scale_columns(U, S, us.d(), n1, k, p, s);
    else
        launch_scale_columns_strided(U, S, us.d(), n1, k, kstride, p, s);
    // Chat_i (n1 x n2) = US_i (n1 x k) * V_i^T: B(kk, n) = V_i[n + kk*n2]
    GemmDesc d;
    d.M = n1; d.N = n2; d.K = k; d.batch = p;
    d.A = us.d(); d.lda = n1; d.strideA = n1 * k;
    d.B = V; d.ldb = n2; d.strideB = n2 * kstride; d.b_nmajor = true;
    d.C = Chat; d.ldc = n1; d.strideC = n1 * n2;
    gemm(d, s);
}

void reconstruct(const double* U, const double* S, const double* V, const double* Q, int64_t n1,
                 int64_t n2, int64_t n3, int64_t p, int64_t k, double* out, cudaStream_t s,
                 int64_t kstride) {
    DeviceBuffer ch(sizeof(double) * n1 * n2 * p);
    core_from_factors(U, S, V, n1, n2, p, k, ch.d(), s, kstride);
    mode3(ch.d(), n1 * n2, p, Q, n3, false, out, 1.0, s);
}

std::array<double, 2> recon_residual(const double* A, int64_t n1, int64_t n2, int64_t n3,
                                     const double* U, const double* S, const double* V,
                                     const double* Q, int64_t p, int64_t k, cudaStream_t s,
                                     int64_t kstride) {
    const int64_t N = n1 * n2;
    StageTimer tm("recon_residual", s, 2.0 * p * N * k + 2.0 * N * p * n3, 8.0 * N * (p + n3));
    DeviceBuffer ch(sizeof(double) * N * p);
    core_from_factors(U, S, V, n1, n2, p, k, ch.d(), s, kstride);
    {
        std::array<double, 2> oz{};
        if (ozaki_recon_residual(A, N, n3, ch.d(), Q, p, oz.data(), s)) return oz;
    }
    GemmDesc d;
    d.M = N; d.N = n3; d.K = p;
    d.A = ch.d(); d.lda = N;
    d.B = Q; d.ldb = n3; d.b_nmajor = true;
    return residual_sums(d, A, N, 0, s);
}

std::array<double, 2> recon_residual_block(const double* A_blk, int64_t n1, int64_t nj, int64_t n3,
                                           int64_t ldA, const double* U, const double* S,
                                           const double* V, int64_t n2, int64_t j0,
                                           const double* Q, int64_t p, int64_t k, cudaStream_t s) {
    // Chat_i restricted to columns [j0, j0+nj): (U_i S_i) V_i[j0:j0+nj, :]^T
    const int64_t Nb = n1 * nj;
    StageTimer tm("recon_residual", s, 2.0 * p * Nb * k + 2.0 * Nb * p * n3, 8.0 * Nb * (p + n3));
    DeviceBuffer us(sizeof(double) * n1 * k * p), ch(sizeof(double) * Nb * p);
    launch_scale_columns(U, S, us.d(), n1, k, p, s);
    {
        GemmDesc d;
        d.M = n1; d.N = nj; d.K = k; d.batch = p;
        d.A = us.d(); d.lda = n1; d.strideA = n1 * k;
        d.B = V + j0; d.ldb = n2; d.strideB = n2 * k; d.b_nmajor = true;
        d.C = ch.d(); d.ldc = n1; d.strideC = Nb;
        gemm(d, s);
    }
    // The block's tube matrix: row i + (j-j0)*n1 is contiguous inside each
    // frontal slice (lateral columns j0.. are adjacent), column stride ldA.
    GemmDesc d;
    d.M = Nb; d.N = n3; d.K = p;
    d.A = ch.d(); d.lda = Nb;
    d.B = Q; d.ldb = n3; d.b_nmajor = true;
    const int64_t ctas = gemm_residual_ctas(d, A_blk, ldA, 0);
    DeviceBuffer part(sizeof(double) * 2 * (ctas + 1));
    gemm_residual(d, A_blk, ldA, 0, part.d(), s);
    double* fin = part.d() + 2 * ctas;
    launch_reduce_pairs(part.d(), ctas, fin, s);
    std::array<double, 2> out{};
    PPC_CUDA_CHECK(cudaMemcpyAsync(out.data(), fin, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    return out;
}

double compress_relative_error(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* U,
                               const double* S, const double* V, const double* Q, int64_t p, int64_t k,
                               const double* est, cudaStream_t s) {
    static const bool identity = !(std::getenv("PPC_RE_IDENTITY") && std::getenv("PPC_RE_IDENTITY")[0] == '0');
    double h[3];
    PPC_CUDA_CHECK(cudaMemcpyAsync(h, est, sizeof(h), cudaMemcpyDeviceToHost, s));
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    if (h[0] == 0.0) fail(PPC_DEGENERATE, "relative_error: reference tensor is zero");
    const double num = (h[0] - h[2]) + h[1];
    if (identity && std::isfinite(num) && num >= 2e-3 * h[0]) return std::sqrt(num) / std::sqrt(h[0]);
    const auto r = recon_residual(A, n1, n2, n3, U, S, V, Q, p, k, s);
    if (r[1] == 0.0) fail(PPC_DEGENERATE, "relative_error: reference tensor is zero");
    return std::sqrt(r[0]) / std::sqrt(r[1]);
}

void tsvdq(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* Q, int64_t p,
           int64_t k, double* U, double* S, double* V, cudaStream_t s, double* slice_sums,
           const OzakiDigits* tdig, const double* a2) {
    const int64_t N = n1 * n2;
    DeviceBuffer ah(sizeof(double) * N * p);
    if (!(tdig && ozaki_mode3_forward(*tdig, N, Q, p, ah.d(), s)))
        mode3(A, N, n3, Q, p, true, ah.d(), 1.0, s);  // decompositions.cpp:65
    {
        StageTimer tm("slice_svd", s, (double)p * std::min(n1, n2) * std::min(n1, n2) * std::max(n1, n2) +
                                          4.0 * p * N * k, 8.0 * p * N);
        // :75-81, with the input check of matrix_kernels.cpp:32
        slice_svd(ah.d(), n1, n2, N, p, k, U, S, V, nullptr, s, "svd");
    }
    if (!slice_sums) return;
    // Eckart-Young through the polish: U_i S_i V_i^T = Ahat_i V_k V_k^T for the
    // orthonormal Rayleigh-Ritz basis V_k (W = Ahat_i V_k = Q R, R = U_r S V_r^T,
    // U = Q U_r, V = V_k V_r), so ||Ahat_i - U_i S_i V_i^T||^2 =
    // ||Ahat_i||^2 - sum_j s_ij^2 and the compress RE^2 is ||A||^2 - sum s^2:
    // no residual pass over Ahat. The s_ij carry ~eps s_i1 each, ~2 eps k ||A||^2
    // on the sum at worst, so it is taken only while RE^2 >= 2e-2 ||A||^2
    // (<= 4e-13 relative in RE); below, the fused residual GEMM runs.
    static const bool sigma_id = !(std::getenv("PPC_RE_SIGMA") && std::getenv("PPC_RE_SIGMA")[0] == '0') &&
                                 !(std::getenv("PPC_RE_IDENTITY") && std::getenv("PPC_RE_IDENTITY")[0] == '0');
    if (a2 && sigma_id) {
        DeviceBuffer part(sizeof(double) * (2 * kReduceBlocks + 2));
        double* fin = part.d() + 2 * kReduceBlocks;
        launch_sumsq_partials(S, nullptr, k * p, part.d(), s);
        launch_reduce_pairs(part.d(), kReduceBlocks, fin, s);
        double h[2];
        PPC_CUDA_CHECK(cudaMemcpyAsync(&h[0], a2, sizeof(double), cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaMemcpyAsync(&h[1], fin + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
        const double num = h[0] - h[1];
        if (std::isfinite(num) && num >= 2e-2 * h[0]) {
            // slice_sums = {0, sum s^2}: compress_relative_error's (||A||^2 -
            // slice_sums[1]) + slice_sums[0] is then ||A||^2 - sum s^2
            PPC_CUDA_CHECK(cudaMemsetAsync(slice_sums, 0, sizeof(double), s));
            PPC_CUDA_CHECK(
                cudaMemcpyAsync(slice_sums + 1, fin + 1, sizeof(double), cudaMemcpyDeviceToDevice, s));
            return;
        }
    }
    slice_residual_sums(ah.d(), n1, n2, p, k, U, S, V, slice_sums, s);
}

void slice_residual_sums(const double* Ah, int64_t n1, int64_t n2, int64_t p, int64_t k, const double* U,
                         const double* S, const double* V, double* out, cudaStream_t s) {
    const int64_t N = n1 * n2;
    StageTimer tm("slice_residual", s, 2.0 * p * N * k, 8.0 * p * N);
    DeviceBuffer us(sizeof(double) * n1 * k * p);
    launch_scale_columns(U, S, us.d(), n1, k, p, s);
    GemmDesc d;
    d.M = n1; d.N = n2; d.K = k; d.batch = p;
    d.A = us.d(); d.lda = n1; d.strideA = n1 * k;
    d.B = V; d.ldb = n2; d.strideB = n2 * k; d.b_nmajor = true;
    // one total (no per-slice sums): the warp-specialized TMA kernel may run it
    const int64_t ctas = gemm_residual_ctas(d, Ah, n1, N);
    DeviceBuffer part(sizeof(double) * 2 * ctas);
    gemm_residual(d, Ah, n1, N, part.d(), s);
    launch_reduce_pairs(part.d(), ctas, out, s);
}

void sweep_errors(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* Q, int64_t pmax,
                  int64_t kmax, const int64_t* ps, int64_t np, const int64_t* ks, int64_t nk, double* re,
                  cudaStream_t s) {
    const int64_t N = n1 * n2;
    DeviceBuffer ah(sizeof(double) * N * pmax), U(sizeof(double) * n1 * kmax * pmax),
        S(sizeof(double) * kmax * pmax), V(sizeof(double) * n2 * kmax * pmax);
    mode3(A, N, n3, Q, pmax, true, ah.d(), 1.0, s);  // all slices at max p
    require_finite(ah.d(), N * pmax, "svd", s);
    {
        StageTimer tm("slice_svd", s);
        slice_svd(ah.d(), n1, n2, N, pmax, kmax, U.d(), S.d(), V.d(), nullptr, s);
    }
    static const bool identity = !(std::getenv("PPC_RE_IDENTITY") && std::getenv("PPC_RE_IDENTITY")[0] == '0');
    double anorm2[2];
    sumsq(A, nullptr, N * n3, anorm2, s);
    if (anorm2[1] == 0.0) fail(PPC_DEGENERATE, "relative_error: reference tensor is zero");
    DeviceBuffer us(sizeof(double) * n1 * kmax * pmax), ch;
    // Eckart-Young through the polish (see tsvdq): RE^2(p, k) = ||A||^2 -
    // sum_{i < p, j < k} s_ij^2 while that stays >= 2e-2 ||A||^2 (host sums of
    // the kmax x pmax singular values, fixed order)
    static const bool sigma_id = identity && !(std::getenv("PPC_RE_SIGMA") && std::getenv("PPC_RE_SIGMA")[0] == '0');
    std::vector<double> sh;
    if (sigma_id) {
        sh.resize((size_t)(kmax * pmax));
        PPC_CUDA_CHECK(cudaMemcpyAsync(sh.data(), S.d(), sizeof(double) * kmax * pmax, cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    for (int64_t ip = 0; ip < np; ++ip) {
        const int64_t p = ps[ip];
        for (int64_t ik = 0; ik < nk; ++ik) {
            const int64_t k = ks[ik];
            if (sigma_id) {
                double s2 = 0.0;
                for (int64_t i = 0; i < p; ++i)
                    for (int64_t j = 0; j < k; ++j) s2 = std::fma(sh[j + i * kmax], sh[j + i * kmax], s2);
                const double num = anorm2[1] - s2;
                if (std::isfinite(num) && num >= 2e-2 * anorm2[1]) {
                    re[ik + ip * nk] = std::sqrt(num) / std::sqrt(anorm2[1]);
                    continue;
                }
            }
            // U(:, :k, i) diag(S(:k, i)) V(:, :k, i)^T for the first p slices
            launch_scale_columns_strided(U.d(), S.d(), us.d(), n1, k, kmax, p, s);
            if (identity) {
                // orthogonal split (as in compress_relative_error): ||A - Ahat_k x3 Q||^2 =
                // (||A||^2 - ||Ahat_p||^2) + sum_i ||Ahat_i - U_i S_i V_i^T||^2, both
                // sums from one fused residual pass over the p slices of Ahat
                StageTimer tm("slice_residual", s, 2.0 * p * N * k, 8.0 * p * N);
                GemmDesc d;
                d.M = n1; d.N = n2; d.K = k; d.batch = p;
                d.A = us.d(); d.lda = n1; d.strideA = n1 * k;
                d.B = V.d(); d.ldb = n2; d.strideB = n2 * kmax; d.b_nmajor = true;
                const int64_t ctas = gemm_residual_ctas(d, ah.d(), n1, N);
                DeviceBuffer part(sizeof(double) * 2 * (ctas + 1));
                gemm_residual(d, ah.d(), n1, N, part.d(), s);
                double* fin = part.d() + 2 * ctas;
                launch_reduce_pairs(part.d(), ctas, fin, s);
                double h[2];
                PPC_CUDA_CHECK(cudaMemcpyAsync(h, fin, sizeof(h), cudaMemcpyDeviceToHost, s));
                PPC_CUDA_CHECK(cudaStreamSynchronize(s));
                const double num = (anorm2[1] - h[1]) + h[0];
                if (std::isfinite(num) && num >= 2e-3 * anorm2[1]) {
                    re[ik + ip * nk] = std::sqrt(num) / std::sqrt(anorm2[1]);
                    continue;
                }
            }
            // small errors: measured directly against A (no cancellation)
            StageTimer tm("recon_residual", s, 2.0 * p * N * k + 2.0 * N * p * n3, 8.0 * N * (p + n3));
            if (!ch.d()) ch = DeviceBuffer(sizeof(double) * N * pmax);
            GemmDesc d;
            d.M = n1; d.N = n2; d.K = k; d.batch = p;
            d.A = us.d(); d.lda = n1; d.strideA = n1 * k;
            d.B = V.d(); d.ldb = n2; d.strideB = n2 * kmax; d.b_nmajor = true;
            d.C = ch.d(); d.ldc = n1; d.strideC = N;
            gemm(d, s);
            GemmDesc r;
            r.M = N; r.N = n3; r.K = p;
            r.A = ch.d(); r.lda = N;
            r.B = Q; r.ldb = n3; r.b_nmajor = true;
            const auto sums = residual_sums(r, A, N, 0, s);
            re[ik + ip * nk] = std::sqrt(sums[0]) / std::sqrt(sums[1]);
        }
    }
}

ErrorParts tsvdq_error(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* U,
                       const double* S, const double* V, const double* Q, int64_t p, int64_t k,
                       cudaStream_t s) {
    const int64_t N = n1 * n2;
    // :97-100 recompute A x3 Q^T and fresh slice SVDs for the tail energies
    DeviceBuffer ah(sizeof(double) * N * p);
    mode3(A, N, n3, Q, p, true, ah.d(), 1.0, s);
    require_finite(ah.d(), N * p, "svd", s);
    DeviceBuffer tail(sizeof(double) * p), tsum(sizeof(double) * 2 * 2);
    {
        DeviceBuffer u(sizeof(double) * n1 * k * p), sv(sizeof(double) * k * p),
            v(sizeof(double) * n2 * k * p);
        slice_svd(ah.d(), n1, n2, N, p, k, u.d(), sv.d(), v.d(), tail.d(), s);
    }
    std::vector<double> th(p);
    PPC_CUDA_CHECK(cudaMemcpyAsync(th.data(), tail.d(), sizeof(double) * p, cudaMemcpyDeviceToHost, s));
    // :51-58 total measured directly against the reconstruction (fused)
    const auto tot = recon_residual(A, n1, n2, n3, U, S, V, Q, p, k, s);
    const auto pr = projection_residual(A, N, n3, Q, p, ah.d(), s);
    double ey = 0.0;
    for (int64_t i = 0; i < p; ++i) ey += th[i];  // decompositions.cpp:41-49 order (slice-major)
    return ErrorParts{std::sqrt(tot[0]), std::sqrt(ey), std::sqrt(pr[0])};
}

void tsvdq2_select(const double* s_all, int64_t r, int64_t p, double gamma, int64_t* multirank) {
    // :137-145 pool of values above 1e-12 * the global maximum
    double gmax = 0.0;
    for (int64_t i = 0; i < p; ++i)
        if (r > 0) gmax = std::max(gmax, s_all[i * r]);
    const double cutoff = 1e-12 * gmax;  // kDefaultRankTol (matrix_kernels.hpp)
    struct Entry {
        double value;
        int64_t slice, pos;
    };
    std::vector<Entry> pool;
    pool.reserve((size_t)(r * p));
    for (int64_t i = 0; i < p; ++i)
        for (int64_t j = 0; j < r; ++j)
            if (s_all[j + i * r] > cutoff) pool.push_back({s_all[j + i * r], i, j});
    // :148-150 descending by value, ties by slice then position
    std::sort(pool.begin(), pool.end(), [](const Entry& a, const Entry& b) {
        if (a.value != b.value) return a.value > b.value;
        if (a.slice != b.slice) return a.slice < b.slice;
        return a.pos < b.pos;
    });
    // :154-167 prefix energy in sorted order decides K
    std::vector<double> cum(pool.size());
    double acc = 0.0;
    for (size_t i = 0; i < pool.size(); ++i) {
        acc += pool[i].value * pool[i].value;
        cum[i] = acc;
    }
    const double total = pool.empty() ? 0.0 : cum.back();
    size_t K = 0;
    if (total > 0.0) {
        const double want = gamma * total;
        while (K < pool.size() && cum[K] < want) ++K;
        ++K;
        K = std::min(K, pool.size());
    }
    for (int64_t i = 0; i < p; ++i) multirank[i] = 0;
    for (size_t i = 0; i < K; ++i) multirank[pool[i].slice] += 1;
}

namespace {

// All r = min(n1,n2) singular triplets of every transform-domain slice
// (decompositions.cpp:31-37 slice_svds).
void full_slice_svds(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* Q, int64_t p,
                     double* U, double* S, double* V, cudaStream_t s) {
    const int64_t N = n1 * n2, r = std::min(n1, n2);
    DeviceBuffer ah(sizeof(double) * N * p);
    mode3(A, N, n3, Q, p, true, ah.d(), 1.0, s);
    require_finite(ah.d(), N * p, "svd", s);
    StageTimer tm("slice_svd", s, (double)p * r * r * std::max(n1, n2), 8.0 * p * N);
    slice_svd(ah.d(), n1, n2, N, p, r, U, S, V, nullptr, s);
}

}  // namespace

void tsvdq2(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* Q, int64_t p,
            double gamma, double* U, double* S, double* V, int64_t* multirank, cudaStream_t s) {
    const int64_t r = std::min(n1, n2);
    full_slice_svds(A, n1, n2, n3, Q, p, U, S, V, s);  // :125-126
    std::vector<double> sh((size_t)(r * p));
    PPC_CUDA_CHECK(cudaMemcpyAsync(sh.data(), S, sizeof(double) * r * p, cudaMemcpyDeviceToHost, s));
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    tsvdq2_select(sh.data(), r, p, gamma, multirank);
    // :178-188 keep the leading multirank[i] triplets of slice i
    DeviceBuffer rk(sizeof(int64_t) * p);
    PPC_CUDA_CHECK(cudaMemcpyAsync(rk.d(), multirank, sizeof(int64_t) * p, cudaMemcpyHostToDevice, s));
    launch_truncate_columns(U, n1, r, p, rk.as<int64_t>(), s);
    launch_truncate_columns(S, 1, r, p, rk.as<int64_t>(), s);
    launch_truncate_columns(V, n2, r, p, rk.as<int64_t>(), s);
    PPC_CUDA_CHECK(cudaStreamSynchronize(s));  // rk and the pageable multirank outlive the copy
}

void tsvdq2_reconstruct(const double* U, const double* S, const double* V, const double* Q,
                        int64_t n1, int64_t n2, int64_t n3, int64_t p, const int64_t* multirank,
                        double* out, cudaStream_t s) {
    const int64_t r = std::min(n1, n2);
    int64_t kmax = 0;
    for (int64_t i = 0; i < p; ++i) kmax = std::max(kmax, multirank[i]);
    reconstruct(U, S, V, Q, n1, n2, n3, p, kmax, out, s, r);
}

ErrorParts tsvdq2_error(const double* A, int64_t n1, int64_t n2, int64_t n3, const double* U,
                        const double* S, const double* V, const double* Q, int64_t p,
                        const int64_t* multirank, cudaStream_t s) {
    const int64_t N = n1 * n2, r = std::min(n1, n2);
    // :205-206 fresh full slice spectra for the tail energies
    std::vector<double> sh((size_t)(r * p));
    {
        DeviceBuffer u(sizeof(double) * n1 * r * p), sv(sizeof(double) * r * p),
            v(sizeof(double) * n2 * r * p);
        full_slice_svds(A, n1, n2, n3, Q, p, u.d(), sv.d(), v.d(), s);
        PPC_CUDA_CHECK(cudaMemcpyAsync(sh.data(), sv.d(), sizeof(double) * r * p, cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    double ey = 0.0;  // decompositions.cpp:41-49 order: slice-major, position ascending
    for (int64_t i = 0; i < p; ++i)
        for (int64_t j = multirank[i]; j < r; ++j) ey += sh[j + i * r] * sh[j + i * r];
    int64_t kmax = 0;
    for (int64_t i = 0; i < p; ++i) kmax = std::max(kmax, multirank[i]);
    const auto tot = recon_residual(A, n1, n2, n3, U, S, V, Q, p, kmax, s, r);
    const auto pr = projection_residual(A, N, n3, Q, p, nullptr, s);
    return ErrorParts{std::sqrt(tot[0]), std::sqrt(ey), std::sqrt(pr[0])};
}

}  // namespace ppc
