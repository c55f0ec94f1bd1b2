// K5b — direct top-p eigensolver for ONE symmetric PSD n x n matrix (the
// data-driven Q's Gram: transforms.cpp:97-115 takes U3 = left singular
// vectors of the mode-3 unfolding, i.e. the top eigenvectors of G = T^T T).
//
// The Chebyshev subspace iteration (subspace.cu) is right for the 128-slice
// batches of the facewise SVD, but for a single 1024 x 1024 Gram it spends
// its time in one-CTA b x b Rayleigh-Ritz eigensolves on a noise plateau
// (~40 ms at cfg5). The direct route here is latency-bound instead:
//   1. Householder tridiagonalization T = H^T G H (LAPACK dsytd2, lower) in
//      ONE persistent cooperative kernel: the matrix lives column-cyclic in
//      the CTAs' shared memory; the owner of column j+1 publishes it before
//      the step-j update, so every CTA rebuilds the next reflector itself and
//      a step needs a single grid barrier (for the p = tau*G*v exchange);
//   2. the top-p eigenvalues of T by Sturm-count bisection, 32-way
//      multisection per warp (one warp per eigenvalue);
//   3. their eigenvectors by inverse iteration on T - lambda I (tridiagonal
//      LU with partial pivoting, deterministic random starts, 3 solves);
//   4. shifted CholQR3 of Z in eigenvalue order (DMMA GEMMs, subspace.cu);
//   5. back-transformation Q = H_0 ... H_{n-3} Z, one warp per column of Z
//      held in registers, reflectors read from L2.
// Every reduction has a fixed order, so Q is bitwise repeatable.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "engine.h"
#include "internal.h"
#include "slice_svd.cuh"

namespace ppc {

namespace {

constexpr int kTrdThreads = 512;
constexpr double kEps = 2.220446049250313e-16;
constexpr double kSafeMin = 2.2250738585072014e-308;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier over co-resident CTAs (cooperative launch) on a monotonic
// arrival counter: barrier number b completes when the counter reaches
// b * nblk, so nobody resets anything on the critical path.
// (A flag per CTA, stored with release and polled by one warp with relaxed
// vector loads and a closing acquire fence, measured slower: 6.3 against
// 4.5 us a step at n = 1024 with 148 CTAs. The arrivals do not serialize in
// L2 the way the same-address atomic model suggests; the second fence costs
// more.)
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblk, unsigned& target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        target += nblk;
        // release: this CTA's writes (ordered before by bar.sync) are visible
        // to whoever acquires the counter; no return value to wait for
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while (ld_acquire(bar) < target) {
        }
    }
    __syncthreads();
}

// Fixed-order block sum (every CTA running the same code on the same data
// gets the same bits): thread-strided partials, then a fixed tree.
// red: 2 x 32 doubles, used alternately (the parity flips per call), so the
// next call's writes never race this call's reads: one barrier per sum.
__device__ __forceinline__ double block_sum(double v, double* red, int& par) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double* r = red + 32 * par;
    par ^= 1;
    if (lane == 0) r[warp] = v;
    __syncthreads();
    double t = lane < nw ? r[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;  // every thread
}

struct TrdParams {
    const double* G;  // n x n, column-major, symmetric
    int n, nblk, cpc;
    double* V;       // n x n: column j = v_j (zeros in rows <= j, 1 in row j+1)
    double* tau;     // n
    double* d;       // n
    double* e;       // n - 1
    double* pg;      // 2 x n  exchanged p = tau * A v, by step parity (a fast CTA
                     //        writes step j+1 while a slow one still reads step j)
    double* colpub;  // 2 x n  published next pivot column, by step parity
    unsigned* bar;   // arrival counter (one per matrix, 128 bytes apart)
    double* Aw;      // hybrid variant: the owned slots < cpc - cps in global memory
                     // (L2), [matrix][CTA][slot][n]; nullptr: all in shared memory
    int cps;         // the last cps slots live in shared memory (hybrid variant):
                     // the highest columns, which stay in the trailing matrix longest
    // batch: matrix b is G + b * strideG; its nblk CTAs are blocks
    // [b * nblk, (b+1) * nblk) and every output above is per matrix
    int64_t strideG;
    int blk;         // the CTA's rank within its matrix (set in the kernel)
    long long* prof; // built with -DPPC_TRD_PROFILE and run with PPC_TRD_PROFILE=1: per-warp
                     // clock sums of the step's phases (else nullptr)
};

constexpr size_t kTrdSmemMax = 200 * 1024;
#ifndef PPC_TRD_KC
#define PPC_TRD_KC 4
#endif
#ifndef PPC_TRD_KU
#define PPC_TRD_KU 2
#endif
constexpr int kTrdKc = PPC_TRD_KC, kTrdKu = PPC_TRD_KU;  // columns per warp at once, row pairs per lane per round

// Reflector of step jj from column jj (xs, rows jj+1..n-1), LAPACK dlarfg:
// computed redundantly by every CTA (same bits everywhere). Writes vn and
// returns tau; the CTA's slice of V(:, jj) and (CTA 0) d, e, tau go out.
__device__ __forceinline__ double make_reflector(const TrdParams& P, int jj, const double* xs, double* vn,
                                                 double* red, int& rpar) {
    const int n = P.n, tid = threadIdx.x, nt = blockDim.x;
    double s2 = 0.0;
    for (int i = jj + 2 + tid; i < n; i += nt) s2 = fma(xs[i], xs[i], s2);
    s2 = block_sum(s2, red, rpar);
    const double alpha = xs[jj + 1];
    double beta, tau, scal;
    if (s2 == 0.0) {
        beta = alpha;
        tau = 0.0;
        scal = 0.0;
    } else {
        beta = -copysign(sqrt(fma(alpha, alpha, s2)), alpha);
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
    }
    for (int i = tid; i < n; i += nt) vn[i] = i <= jj ? 0.0 : (i == jj + 1 ? 1.0 : xs[i] * scal);
    if (P.blk == 0 && tid == 0) {
        P.d[jj] = xs[jj];
        P.e[jj] = beta;
        P.tau[jj] = tau;
    }
    // V(:, jj): CTA b stores rows [b*ch, (b+1)*ch)
    const int ch = (n + P.nblk - 1) / P.nblk;
    const int r0 = P.blk * ch;
    for (int i = r0 + tid; i < min(n, r0 + ch); i += nt)
        P.V[(size_t)jj * n + i] = i <= jj ? 0.0 : (i == jj + 1 ? 1.0 : xs[i] * scal);
    return tau;
}

// Slots [ta, tb) of the owned columns, stored at base + (t - ta) * n (GM: in
// the global working copy, read and written through L2 with ld/st.cg; else in
// shared memory). A warp takes KC of its columns at once over the same rows,
// KU row pairs of each per lane per round: v, w and v' are read from shared
// memory once per KC columns (a column at a time spent 24 of every 40 bytes
// of shared-memory traffic on them), and KC * KU loads are in flight (from L2
// a column at a time paid one round trip per 256 rows). Every column's
// products keep the row order of a lane, so the bits do not depend on KC, KU
// or on where the column lives.
template <bool GM, int KC, int KU>
__device__ __forceinline__ void update_range(const TrdParams& P, double* base, int ta, int tb, int j,
                                             const double* vs, const double* ws, const double* vn, double taun,
                                             double* pgo, double* cp, bool by_slot) {
    const int n = P.n, nblk = P.nblk, blk = P.blk;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int i0 = (j + 1) & ~1;
    for (int t0 = ta + warp; t0 < tb; t0 += KC * nw) {
        bool ok[KC];
        double vc[KC], wc[KC], acc[KC];
        bool any = false;
#pragma unroll
        for (int q = 0; q < KC; ++q) {
            const int t = t0 + q * nw;
            const int c = blk + t * nblk;
            ok[q] = t < tb && c > j && c < n;  // warp-uniform
            any |= ok[q];
            vc[q] = ok[q] ? vs[c] : 0.0;
            wc[q] = ok[q] ? ws[c] : 0.0;
            acc[q] = 0.0;
        }
        if (!any) continue;
        double* a0 = base + (size_t)(t0 - ta) * n;
        const size_t astep = (size_t)nw * n;
        for (int ib = i0 + 2 * lane; ib < n; ib += 64 * KU) {
            double2 av[KC][KU];
#pragma unroll
            for (int q = 0; q < KC; ++q)
#pragma unroll
                for (int u = 0; u < KU; ++u) {
                    const int i = ib + 64 * u;
                    const double2* src = reinterpret_cast<const double2*>(a0 + q * astep + i);
                    av[q][u] = ok[q] && i < n ? (GM ? __ldcg(src) : *src) : make_double2(0.0, 0.0);
                }
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                const int i = ib + 64 * u;
                if (i >= n) break;
                const double2 v2 = *reinterpret_cast<const double2*>(vs + i);
                const double2 w2 = *reinterpret_cast<const double2*>(ws + i);
                const double2 n2 = vn ? *reinterpret_cast<const double2*>(vn + i) : make_double2(0.0, 0.0);
#pragma unroll
                for (int q = 0; q < KC; ++q) {
                    if (!ok[q]) continue;
                    double2 nv;
                    nv.x = fma(-w2.x, vc[q], fma(-v2.x, wc[q], av[q][u].x));
                    nv.y = fma(-w2.y, vc[q], fma(-v2.y, wc[q], av[q][u].y));
                    double2* dst = reinterpret_cast<double2*>(a0 + q * astep + i);
                    if (GM) __stcg(dst, nv);
                    else *dst = nv;
                    if (vn) {
                        acc[q] = fma(nv.x, n2.x, acc[q]);
                        acc[q] = fma(nv.y, n2.y, acc[q]);
                    }
                    if (blk + (t0 + q * nw) * nblk == j + 2) *reinterpret_cast<double2*>(cp + i) = nv;
                }
            }
        }
        if (vn) {
#pragma unroll
            for (int q = 0; q < KC; ++q) {
                if (!ok[q]) continue;
                double r = acc[q];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
                const int t = t0 + q * nw, c = blk + t * nblk;
                if (lane == 0 && c > j + 1) pgo[by_slot ? t : c] = taun * r;
            }
        }
    }
}

// One pass over the owned columns c > j: the step-j rank-2 update
// A(j+1:, c) -= v w_c + w v_c, fused with the step-(j+1) products
// p_c = tau' A(j+2:, c)^T v' of the updated columns (vn == nullptr: update
// only). Two rows per lane per iteration from an even start (v, w and v' are
// zero in rows <= j, so the extra row is left unchanged); the owner of column
// j+2 publishes it as it goes. The products go to pgo[c] (pgo[slot] with
// by_slot) and the published column to cp.
__device__ __forceinline__ void update_pass(const TrdParams& P, double* A, int j, const double* vs,
                                            const double* ws, const double* vn, double taun, double* pgo,
                                            double* cp, bool by_slot) {
    const int cpc = P.cpc;
    const int t1 = P.Aw ? cpc - P.cps : 0;  // slots [0, t1) in L2, [t1, cpc) in shared memory
    if (t1 > 0) update_range<true, kTrdKc, kTrdKu>(P, P.Aw, 0, t1, j, vs, ws, vn, taun, pgo, cp, by_slot);
    if (t1 < cpc) {
        // few columns per warp (a single matrix spread over every SM): one at a
        // time, or the chunk's empty columns would only cost predicates
        if (cpc - t1 <= (int)(blockDim.x >> 5))
            update_range<false, 1, 4>(P, A, t1, cpc, j, vs, ws, vn, taun, pgo, cp, by_slot);
        else
            update_range<false, kTrdKc, kTrdKu>(P, A, t1, cpc, j, vs, ws, vn, taun, pgo, cp, by_slot);
    }
}

// Column c is owned by CTA c % nblk, slot c / nblk.
template <int NT>
__global__ void __launch_bounds__(NT, 1) sytrd_kernel(TrdParams P0) {
    extern __shared__ __align__(16) double sm[];
    // this CTA's matrix and rank, and the matrix's slices of every array
    TrdParams P = P0;
    const int mat = blockIdx.x / P0.nblk;
    P.blk = blockIdx.x % P0.nblk;
    {
        const size_t n0 = (size_t)P0.n;
        P.G += (size_t)mat * P0.strideG;
        P.V += (size_t)mat * n0 * n0;
        P.tau += (size_t)mat * n0;
        P.d += (size_t)mat * n0;
        P.e += (size_t)mat * n0;
        P.pg += (size_t)mat * 2 * n0;
        P.colpub += (size_t)mat * 2 * n0;
        P.bar += (size_t)mat * 32;
    }
    const int n = P.n, nblk = P.nblk, cpc = P.cpc, blk = P.blk;
    // cpc x n (slot t = column blk + t*nblk): the last cps slots in shared
    // memory, the first cpc - cps (hybrid variant) in this CTA's slice of the
    // global working copy
    const int t1 = P.Aw ? cpc - P.cps : 0;  // first shared-memory slot
    if (P.Aw) P.Aw += ((size_t)mat * nblk + blk) * (size_t)t1 * n;
    double* A = sm;
    double* vs = A + (size_t)(cpc - t1) * n;  // reflector of step j
    double* vn = vs + n;               // reflector of step j+1
    double* ws = vn + n;               // w = p - K v
    double* xs = ws + n;               // pivot column
    __shared__ double red[64];
    int rpar = 0;
    const int tid = threadIdx.x, nt = blockDim.x;
    unsigned target = 0;

    for (int t = 0; t < cpc; ++t) {
        const int c = blk + t * nblk;
        if (c < n)
            for (int i = tid; i < n; i += nt)
                (t >= t1 ? A + (size_t)(t - t1) * n : P.Aw + (size_t)t * n)[i] = P.G[(size_t)c * n + i];
    }
    for (int i = tid; i < n; i += nt) {
        xs[i] = P.G[i];
        ws[i] = 0.0;
    }
    __syncthreads();
    // prologue: reflector 0, its products, column 1 published (an update
    // with v = w = 0 leaves A unchanged)
    double tau = make_reflector(P, 0, xs, vn, red, rpar);
    for (int i = tid; i < n; i += nt) vs[i] = 0.0;
    __syncthreads();
    update_pass(P, A, -1, vs, ws, vn, tau, P.pg, P.colpub, false);

    for (int j = 0; j <= n - 3; ++j) {
        {
            double* t = vs;  // the step-j reflector is the one just built
            vs = vn;
            vn = t;
        }
#ifdef PPC_TRD_PROFILE
        long long c0 = 0, c1 = 0, c2 = 0, c3 = 0;
        if (P.prof) c0 = clock64();
#endif
        grid_barrier(P.bar, (unsigned)nblk, target);
#ifdef PPC_TRD_PROFILE
        if (P.prof) c1 = clock64();
#endif
        // ---- p and the published column j+1 (both written before the barrier)
        const double* pg = P.pg + (size_t)(j & 1) * n;
        const double* cp = P.colpub + (size_t)(j & 1) * n;
        double pv = 0.0;
        for (int i = j + 1 + tid; i < n; i += nt) {
            const double p = __ldcg(pg + i);
            ws[i] = p;
            xs[i] = __ldcg(cp + i);
            pv = fma(p, vs[i], pv);
        }
        const double K = 0.5 * tau * block_sum(pv, red, rpar);
        // w = p - K v and the pivot column j+1 after the step-j update, in one
        // pass (w(j+1) recomputed from p(j+1): no barrier between the two)
        {
            const double vc = vs[j + 1], wc = fma(-K, vc, __ldcg(pg + j + 1));
            for (int i = j + 1 + tid; i < n; i += nt) {
                const double w = fma(-K, vs[i], ws[i]);
                ws[i] = w;
                xs[i] = fma(-w, vc, fma(-vs[i], wc, xs[i]));
            }
        }
        if (tid == 0) ws[j] = 0.0;  // rows <= j of w stay zero (read by the paired-row pass)
        __syncthreads();
#ifdef PPC_TRD_PROFILE
        if (P.prof) c2 = clock64();
#endif
        if (j + 1 <= n - 3) {
            const double taun = make_reflector(P, j + 1, xs, vn, red, rpar);
            __syncthreads();
#ifdef PPC_TRD_PROFILE
            if (P.prof) c3 = clock64();
#endif
            update_pass(P, A, j, vs, ws, vn, taun, P.pg + (size_t)((j + 1) & 1) * n,
                        P.colpub + (size_t)((j + 1) & 1) * n, false);
            tau = taun;
#ifdef PPC_TRD_PROFILE
            if (P.prof && (tid & 31) == 0) {  // per warp: barrier wait, p/w pass, reflector, update
                long long* q = P.prof + ((size_t)blockIdx.x * (nt >> 5) + (tid >> 5)) * 4;
                q[0] += c1 - c0;
                q[1] += c2 - c1;
                q[2] += c3 - c2;
                q[3] += clock64() - c3;
            }
#endif
        } else {
            update_pass(P, A, j, vs, ws, nullptr, 0.0, nullptr, P.colpub + (size_t)((j + 1) & 1) * n, false);
        }
        // (the next step's grid barrier opens with a block barrier)
    }
    // trailing 2 x 2 block: columns n-2 and n-1 are final in their owners
    for (int t = 0; t < cpc; ++t) {
        const int c = blk + t * nblk;
        if (tid == 0 && c == n - 2) {
            const double* a = t >= t1 ? A + (size_t)(t - t1) * n : P.Aw + (size_t)t * n;
            P.d[n - 2] = a[n - 2];
            P.e[n - 2] = a[n - 1];
            P.tau[n - 2] = 0.0;
        }
        if (tid == 0 && c == n - 1) {
            const double* a = t >= t1 ? A + (size_t)(t - t1) * n : P.Aw + (size_t)t * n;
            P.d[n - 1] = a[n - 1];
            P.tau[n - 1] = 0.0;
        }
    }
}

// Number of eigenvalues of T below x (Sturm sequence, LAPACK dlaneg-style
// pivot guard).
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x,
                                           double pivmin) {
    double q = d[0] - x;
    if (fabs(q) <= pivmin) q = -pivmin;
    int c = q < 0.0;
    for (int i = 1; i < n; ++i) {
        q = d[i] - x - e2[i - 1] / q;
        if (fabs(q) <= pivmin) q = -pivmin;
        c += q < 0.0;
    }
    return c;
}

// One CTA per wanted eigenvalue m (0 = largest): NT-way
// multisection, every thread one Sturm count per round (~7 bits a round).
// NT = 256 for a few eigenvalues (latency: 8 bits a round); 64 when a batch
// brings hundreds (work: the SMs are full either way).
// kl CTAs per matrix compute eigenvalues m0 .. m0 + kl - 1 of its k wanted
// (kl = k, m0 = 0 for all of them; a subrange for the sharded eigensolve:
// every eigenvalue comes out bitwise the same either way).
template <int NT>
__global__ void __launch_bounds__(NT) bisect_top_kernel(const double* __restrict__ dg,
                                                                 const double* __restrict__ eg, int n, int k,
                                                                 double* __restrict__ lam,
                                                                 double* __restrict__ bounds, int kl, int m0) {
    extern __shared__ __align__(16) double sh[];
    {  // matrix blockIdx.x / kl of the batch
        const int mat = blockIdx.x / kl;
        dg += (size_t)mat * n;
        eg += (size_t)mat * n;
        lam += (size_t)mat * k;
        bounds += (size_t)mat * 2;
    }
    double* d = sh;
    double* e2 = sh + n;
    __shared__ double s_gl[NT / 32], s_gu[NT / 32], s_em[NT / 32];
    __shared__ int s_first[NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
    // Gershgorin interval and the pivot floor (fixed order: same in every CTA)
    double gl = 1e308, gu = -1e308, em = 0.0;
    for (int i = tid; i < n; i += NT) {
        const double di = dg[i];
        const double el = i > 0 ? fabs(eg[i - 1]) : 0.0, er = i < n - 1 ? fabs(eg[i]) : 0.0;
        d[i] = di;
        e2[i] = er * er;
        gl = fmin(gl, di - el - er);
        gu = fmax(gu, di + el + er);
        em = fmax(em, er * er);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
        gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
        em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
    }
    if (lane == 0) {
        s_gl[warp] = gl;
        s_gu[warp] = gu;
        s_em[warp] = em;
    }
    __syncthreads();
    gl = s_gl[0];
    gu = s_gu[0];
    em = s_em[0];
    for (int w = 1; w < nw; ++w) {
        gl = fmin(gl, s_gl[w]);
        gu = fmax(gu, s_gu[w]);
        em = fmax(em, s_em[w]);
    }
    const double tnorm = fmax(fabs(gl), fabs(gu));
    const double pivmin = kSafeMin * fmax(1.0, em);
    gl -= 2.0 * kEps * tnorm * n + 2.0 * pivmin;
    gu += 2.0 * kEps * tnorm * n + 2.0 * pivmin;
    const double atol = kEps * tnorm;
    const int m = m0 + (int)(blockIdx.x % kl);  // eigenvalue of matrix blockIdx.x / kl
    const int want = n - m;  // invariant: count(hi) >= want > count(lo)
    double lo = gl, hi = gu;
    for (int it = 0; it < 40; ++it) {
        if (hi - lo <= fmax(2.0 * kEps * fmax(fabs(lo), fabs(hi)), atol)) break;
        const double x = lo + (hi - lo) * (double)(tid + 1) / (double)(NT + 1);
        const int c = sturm_count(d, e2, n, x, pivmin);
        const unsigned ge = __ballot_sync(0xffffffffu, c >= want);
        if (lane == 0) s_first[warp] = ge ? warp * 32 + __ffs(ge) - 1 : NT;
        __syncthreads();
        int first = NT;
        for (int w = 0; w < nw; ++w) first = min(first, s_first[w]);
        const double h = (double)(hi - lo);
        const double l0 = lo;
        if (first < NT) hi = l0 + h * (double)(first + 1) / (double)(NT + 1);
        if (first > 0) lo = l0 + h * (double)first / (double)(NT + 1);
        __syncthreads();
    }
    if (tid == 0) {
        lam[m] = 0.5 * (lo + hi);
        if (bounds && blockIdx.x % kl == 0) {  // the same values in every CTA of the matrix
            bounds[0] = tnorm;
            bounds[1] = pivmin;
        }
    }
}

__device__ __forceinline__ double hash_unit(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return (double)(z >> 11) * 0x1.0p-52 - 1.0;  // [-1, 1)
}

// Inverse iteration, one CTA (one warp) per eigenvalue: LU with partial
// pivoting of T - lambda I (dlagtf layout: U diagonal u0, superdiagonals
// u1, u2, unit-L multipliers lm, pivot flags) by lane 0 in shared memory,
// three solves from a deterministic random start with max-norm scaling in
// between; the warp loads T, draws the start and normalizes. Pivots below
// eps*||T|| are raised to it (dlagts job = -1).
// (kl, m0 as for bisect_top_kernel: Z holds the kl columns m0 .. m0 + kl - 1)
__global__ void inverse_iteration_kernel(const double* __restrict__ dg, const double* __restrict__ eg,
                                         int n, int k, const double* __restrict__ lam,
                                         const double* __restrict__ bounds, double* __restrict__ Z, int kl,
                                         int m0) {
    {  // matrix blockIdx.x / kl of the batch
        const int mat = blockIdx.x / kl;
        dg += (size_t)mat * n;
        eg += (size_t)mat * n;
        lam += (size_t)mat * k;
        bounds += (size_t)mat * 2;
        Z += (size_t)mat * n * kl;
    }
    extern __shared__ __align__(16) double sh[];
    double* d = sh;
    double* e = d + n;
    double* u0 = e + n;
    double* u1 = u0 + n;
    double* u2 = u1 + n;
    double* lm = u2 + n;
    double* x = lm + n;
    unsigned char* pv = reinterpret_cast<unsigned char*>(x + n);
    __shared__ double s_sc;
    const int m = m0 + (int)(blockIdx.x % kl), lane = threadIdx.x;
    const double l = lam[m];
    const double pert = kEps * fmax(bounds[0], kSafeMin);
    for (int i = lane; i < n; i += 32) {
        d[i] = dg[i] - l;
        e[i] = i < n - 1 ? eg[i] : 0.0;
        x[i] = hash_unit(((uint64_t)m << 32) ^ (uint64_t)i ^ 0x7a11d1a6ULL);
    }
    __syncwarp();
    if (lane == 0) {
        double a0 = d[0], a1 = e[0];
        for (int i = 0; i < n - 1; ++i) {
            const double sub = e[i], dn = d[i + 1], en = e[i + 1];
            if (fabs(a0) >= fabs(sub)) {
                double piv = a0;
                if (fabs(piv) < pert) piv = piv >= 0.0 ? pert : -pert;
                const double mult = sub / piv;
                u0[i] = piv;
                u1[i] = a1;
                u2[i] = 0.0;
                lm[i] = mult;
                pv[i] = 0;
                a0 = fma(-mult, a1, dn);
                a1 = en;
            } else {
                const double mult = a0 / sub;
                u0[i] = sub;
                u1[i] = dn;
                u2[i] = en;
                lm[i] = mult;
                pv[i] = 1;
                a0 = fma(-mult, dn, a1);
                a1 = -mult * en;
            }
        }
        if (fabs(a0) < pert) a0 = a0 >= 0.0 ? pert : -pert;
        u0[n - 1] = a0;
        u1[n - 1] = 0.0;
        u2[n - 1] = 0.0;
        for (int i = 0; i < n; ++i) u0[i] = 1.0 / u0[i];  // reciprocals for the solves
    }
    for (int it = 0; it < 3; ++it) {
        if (lane == 0) {
            double bi = x[0];
            for (int i = 0; i < n - 1; ++i) {
                double bn = x[i + 1];
                if (pv[i]) {
                    const double t = bi;
                    bi = bn;
                    bn = t;
                }
                x[i] = bi;
                bi = fma(-lm[i], bi, bn);
            }
            x[n - 1] = bi;
            double xn1 = 0.0, xn2 = 0.0, mx = 0.0;
            for (int i = n - 1; i >= 0; --i) {
                const double v = fma(-u2[i], xn2, fma(-u1[i], xn1, x[i])) * u0[i];
                x[i] = v;
                xn2 = xn1;
                xn1 = v;
                mx = fmax(mx, fabs(v));
            }
            s_sc = mx > 0.0 ? 1.0 / mx : 1.0;
        }
        __syncwarp();
        const double sc = s_sc;
        for (int i = lane; i < n; i += 32) x[i] *= sc;
        __syncwarp();
    }
    double nrm = 0.0;
    for (int i = lane; i < n; i += 32) nrm = fma(x[i], x[i], nrm);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
    for (int i = lane; i < n; i += 32) Z[(size_t)(m - m0) * n + i] = x[i] * inv;
}

// Q = H_0 H_1 ... H_{n-3} Z. The reflectors go in chunks of kBtChunk,
// last-first; a chunk H_jl ... H_jh (jh applied first) is one compact-WY
// block I - V T V^T (LAPACK dlarft, forward: V = [v_jl .. v_jh], T upper
// triangular), whose T factors are built beforehand by wy_t_kernel. Then
// one warp per column of Z, held in registers (lane l owns row pairs
// 2l + 64 s): d = V^T z in one pass (kBtChunk independent sums), y = T d,
// z -= V y in a second pass. The CTA streams V chunks and T through shared
// memory with cp.async, double-buffered.
constexpr int kBtChunk = 8;
constexpr int kBtWarps = 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// T of chunk c (rows/cols r = 0..cnt-1 <-> reflector jl + r): T(r,r) = tau,
// T(0:r, r) = -tau_r T(0:r, 0:r) V(:, 0:r)^T v_r. One CTA per chunk.
__global__ void wy_t_kernel(const double* __restrict__ V, const double* __restrict__ tau, int n, int nchunks,
                            double* __restrict__ Tout) {
    __shared__ double S[kBtChunk][kBtChunk];
    __shared__ double T[kBtChunk][kBtChunk];
    {  // matrix blockIdx.x / nchunks of the batch
        const size_t mat = blockIdx.x / nchunks;
        V += mat * n * n;
        tau += mat * n;
        Tout += mat * nchunks * kBtChunk * kBtChunk;
    }
    const int c = blockIdx.x % nchunks, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int jtop = n - 3;
    const int j1 = jtop - c * kBtChunk;
    const int cnt = min(kBtChunk, j1 + 1);
    const int jl = j1 - cnt + 1;
    for (int q = warp; q < cnt * cnt; q += nw) {
        const int a = q / cnt, b = q % cnt;
        if (a >= b) continue;
        const double* va = V + (size_t)(jl + a) * n;
        const double* vb = V + (size_t)(jl + b) * n;
        double acc = 0.0;
        for (int i = lane; i < n; i += 32) acc = fma(va[i], vb[i], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) S[a][b] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int r = 0; r < kBtChunk; ++r)
            for (int q = 0; q < kBtChunk; ++q) T[q][r] = 0.0;
        for (int r = 0; r < cnt; ++r) {
            const double tr = tau[jl + r];
            T[r][r] = tr;
            for (int q = 0; q < r; ++q) {
                double acc = 0.0;
                for (int u = q; u < r; ++u) acc = fma(T[q][u], S[u][r], acc);
                T[q][r] = -tr * acc;
            }
        }
        double* out = Tout + (size_t)c * kBtChunk * kBtChunk;
        for (int r = 0; r < kBtChunk; ++r)
            for (int q = 0; q < kBtChunk; ++q) out[q * kBtChunk + r] = T[q][r];  // row-major T(q, r)
    }
}

template <int NS, bool FULL>  // NS doubles per lane (NS/2 row pairs)
__global__ void __launch_bounds__(32 * kBtWarps) back_transform_kernel(const double* __restrict__ V,
                                                                       const double* __restrict__ Tg, int n,
                                                                       int k, double* __restrict__ Z) {
    extern __shared__ __align__(16) double sv[];  // 2 x (kBtChunk x n + kBtChunk^2)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int per_mat = (k + kBtWarps - 1) / kBtWarps;  // CTAs per matrix of the batch
    {
        const size_t mat = blockIdx.x / per_mat;
        const size_t nch = (size_t)(n - 3 + kBtChunk) / kBtChunk;
        V += mat * n * n;
        Tg += mat * nch * kBtChunk * kBtChunk;
        Z += mat * n * k;
    }
    const int col = (blockIdx.x % per_mat) * kBtWarps + warp;
    const bool live = col < k;
    const size_t bufsz = (size_t)kBtChunk * n + kBtChunk * kBtChunk;
    double z[NS];
    double* zc = Z + (size_t)(live ? col : 0) * n;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int i = 2 * lane + 64 * (s >> 1) + (s & 1);
        z[s] = (live && (FULL || i < n)) ? zc[i] : 0.0;
    }
    const int jtop = n - 3;
    const int nchunks = (jtop + kBtChunk) / kBtChunk;
    __shared__ __align__(8) uint64_t full[2];
    // one thread streams a chunk: its cnt reflectors (rows from the first
    // 16-byte-aligned one past the zeros) and T, by the bulk-copy engine
    auto load_chunk = [&](int c, int buf) {
        const int j1 = jtop - c * kBtChunk;
        const int cnt = min(kBtChunk, j1 + 1);
        const int jl = j1 - cnt + 1;
        double* dst = sv + (size_t)buf * bufsz;
        const int r0 = (jl + 1) & ~1;  // rows < r0 are zero in every reflector of the chunk
        const uint32_t rb = (uint32_t)(n - r0) * 8u;
        mbar_expect_tx(&full[buf], cnt * rb + kBtChunk * kBtChunk * 8u);
        for (int r = 0; r < cnt; ++r) bulk_g2s(dst + (size_t)r * n + r0, V + (size_t)(jl + r) * n + r0, rb, &full[buf]);
        bulk_g2s(dst + (size_t)kBtChunk * n, Tg + (size_t)c * kBtChunk * kBtChunk, kBtChunk * kBtChunk * 8u,
                 &full[buf]);
    };
    // rows below the chunk's first nonzero row are never copied: zero them once
    for (size_t q = tid; q < 2 * bufsz; q += 32 * kBtWarps) sv[q] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes before bulk copies
    if (tid == 0) {
        mbar_init(&full[0]);
        mbar_init(&full[1]);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        load_chunk(0, 0);
        if (nchunks > 1) load_chunk(1, 1);
    }
    for (int c = 0; c < nchunks; ++c) {
        mbar_wait(&full[c & 1], (uint32_t)((c >> 1) & 1));
        const int j1 = jtop - c * kBtChunk;
        const int cnt = min(kBtChunk, j1 + 1);
        const double* vb = sv + (size_t)(c & 1) * bufsz;
        const double* T = vb + (size_t)kBtChunk * n;
        double d[kBtChunk];
#pragma unroll
        for (int r = 0; r < kBtChunk; ++r) {
            d[r] = 0.0;
            if (r < cnt) {
                const double* v = vb + (size_t)r * n;
#pragma unroll
                for (int s = 0; s < NS; s += 2) {
                    const int i = 2 * lane + 64 * (s >> 1);
                    if (FULL || i < n) {
                        const double2 v2 = *reinterpret_cast<const double2*>(v + i);
                        d[r] = fma(v2.x, z[s], d[r]);
                        d[r] = fma(v2.y, z[s + 1], d[r]);
                    }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int r = 0; r < kBtChunk; ++r) d[r] += __shfl_xor_sync(0xffffffffu, d[r], o);
        double y[kBtChunk];
#pragma unroll
        for (int q = 0; q < kBtChunk; ++q) {
            double acc = 0.0;
#pragma unroll
            for (int r = q; r < kBtChunk; ++r) acc = fma(T[q * kBtChunk + r], d[r], acc);
            y[q] = acc;  // T rows/cols past cnt are zero
        }
#pragma unroll
        for (int r = 0; r < kBtChunk; ++r) {
            if (r < cnt) {
                const double* v = vb + (size_t)r * n;
#pragma unroll
                for (int s = 0; s < NS; s += 2) {
                    const int i = 2 * lane + 64 * (s >> 1);
                    if (FULL || i < n) {
                        const double2 v2 = *reinterpret_cast<const double2*>(v + i);
                        z[s] = fma(-y[r], v2.x, z[s]);
                        z[s + 1] = fma(-y[r], v2.y, z[s + 1]);
                    }
                }
            }
        }
        __syncthreads();  // buffer c & 1 is refilled by the next-but-one chunk
        if (tid == 0 && c + 2 < nchunks) load_chunk(c + 2, c & 1);
    }
    if (live) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const int i = 2 * lane + 64 * (s >> 1) + (s & 1);
            if (FULL || i < n) zc[i] = z[s];
        }
    }
}

template <int NS>
void launch_back_transform(const double* V, const double* tau, int n, int k, int batch, double* Z, double* Tws,
                           cudaStream_t s) {
    const int nchunks = (n - 3 + kBtChunk) / kBtChunk;
    wy_t_kernel<<<(unsigned)(nchunks * batch), 128, 0, s>>>(V, tau, n, nchunks, Tws);
    count_launch();
    check_launch("wy_t");
    const size_t smem = 2 * ((size_t)kBtChunk * n + kBtChunk * kBtChunk) * sizeof(double);
    const unsigned grid = (unsigned)(((k + kBtWarps - 1) / kBtWarps) * batch);
    if (n == 32 * NS) {
        PPC_CUDA_CHECK(cudaFuncSetAttribute(back_transform_kernel<NS, true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        back_transform_kernel<NS, true><<<grid, 32 * kBtWarps, smem, s>>>(V, Tws, n, k, Z);
    } else {
        PPC_CUDA_CHECK(cudaFuncSetAttribute(back_transform_kernel<NS, false>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        back_transform_kernel<NS, false><<<grid, 32 * kBtWarps, smem, s>>>(V, Tws, n, k, Z);
    }
}

size_t trd_smem(int n, int cpc) { return ((size_t)cpc * n + 4 * (size_t)n) * sizeof(double); }

// CTAs per matrix and owned columns per CTA: a wave of `per_wave` matrices
// runs in one cooperative launch, one CTA per SM, every owned column in
// shared memory (the update pass streams each column once per step: from
// L2 it would be ~1000x the matrix per reduction).
struct TrdPlan {
    int nblk = 0, cpc = 0, per_wave = 0;
};
// Batches that would need more than one wave with every column in shared
// memory (cfg3: 32 Grams of order 512 at 13 CTAs each = 3 waves) run in ONE
// wave with the owned columns in a global working copy instead (L2-resident:
// 64 MB at cfg3): the step latency chain is paid once, not once per wave.
TrdPlan trd_plan_gmem(int64_t n, int64_t batch) {
    TrdPlan t;
    const int sms = ctx().sms;
    if (batch < 2 || batch > sms) return t;
    t.per_wave = (int)batch;
    t.nblk = (int)std::min<int64_t>(sms / batch, n);
    t.cpc = (int)((n + t.nblk - 1) / t.nblk);
    return t;
}

TrdPlan trd_plan(int64_t n, int64_t batch) {
    TrdPlan t;
    const int sms = ctx().sms;
    int nmin = 1;  // fewest CTAs per matrix that fit
    while (nmin <= sms && nmin <= n && trd_smem((int)n, (int)((n + nmin - 1) / nmin)) > kTrdSmemMax) ++nmin;
    if (nmin > sms || nmin > n || batch < 1) return t;
    t.per_wave = (int)std::min<int64_t>(batch, sms / nmin);
    // waves of equal size, then the SMs spread over the wave's matrices
    const int64_t waves = (batch + t.per_wave - 1) / t.per_wave;
    t.per_wave = (int)((batch + waves - 1) / waves);
    t.nblk = (int)std::min<int64_t>(sms / t.per_wave, n);
    // (fewer CTAs with more columns each do not make the step cheaper: 3.4-3.6 us
    // at n = 224 with 148, 56, 28 or 14 CTAs; the barrier's cost is its chain of
    // L2 round trips, not the number of arrivals)
    t.cpc = (int)((n + t.nblk - 1) / t.nblk);
    return t;
}

}  // namespace

bool tridiag_eig_preferred(int64_t n, int64_t p, int64_t batch) {
    if (!tridiag_eig_eligible(n, p, batch)) return false;
    // ~3-5 us a reduction step whatever the size (a latency chain): worth it
    // while the waves' steps stay within cfg3's 3 x 512
    const TrdPlan t = trd_plan(n, batch);
    const int64_t waves = (batch + t.per_wave - 1) / t.per_wave;
    return waves * n <= 1600;
}

bool tridiag_eig_eligible(int64_t n, int64_t p, int64_t batch) {
    if (n < 3 || n > 1536 || (n & 1) || p < 1 || p > 160 || p > n || batch < 1) return false;
    static const bool off = std::getenv("PPC_TRIDIAG_EIG") && std::atoi(std::getenv("PPC_TRIDIAG_EIG")) == 0;
    if (off) return false;
    return trd_plan(n, batch).nblk >= 1;
}

void tridiag_eig_top(const double* G, int64_t n64, int64_t k64, double* Q, double* lambda, cudaStream_t s) {
    tridiag_eig_top_batched(G, n64, n64 * n64, 1, k64, Q, lambda, s);
}

namespace {

// Householder tridiagonalization of `batch` matrices in waves (sytrd_kernel):
// V (n x n x batch), tau, d, e (n x batch).
void run_sytrd(const double* G, int n, int64_t strideG, int batch, double* V, double* tau, double* d, double* e,
               cudaStream_t s) {
    TrdPlan t = trd_plan(n, batch);
    static const bool no_gmem = std::getenv("PPC_TRD_GMEM") && std::getenv("PPC_TRD_GMEM")[0] == '0';
    const bool gmem = !no_gmem && t.per_wave < batch && trd_plan_gmem(n, batch).nblk >= 1;
    if (gmem) t = trd_plan_gmem(n, batch);
    const int nblk = t.nblk, cpc = t.cpc;
    // hybrid (off by default, PPC_TRD_HYBRID_KB = shared memory for the slots):
    // the last cps slots of every CTA (its highest columns, which stay in the
    // trailing matrix longest) in shared memory, the rest in L2. Measured at
    // cfg3 with 40% of the slots in shared memory: no faster than everything in
    // L2 (8.0-8.2 ms a step either way). The update pass moves every trailing
    // element through the SM's load/store path once in and once out wherever
    // it lives; a per-warp clock profile (-DPPC_TRD_PROFILE) puts 55% of the
    // kernel there, 24% in the grid barrier, 10% each in the p/w pass and
    // the reflector.
    static const int hyb_kb = std::getenv("PPC_TRD_HYBRID_KB") ? std::atoi(std::getenv("PPC_TRD_HYBRID_KB")) : 0;
    int cps = cpc;
    if (gmem) {
        const int64_t room = (int64_t)hyb_kb * 1024 - (int64_t)trd_smem(n, 0);
        cps = (int)std::max<int64_t>(0, std::min<int64_t>(cpc, room / ((int64_t)n * (int64_t)sizeof(double))));
    }
    const size_t smem = trd_smem(n, cps);
    const size_t B = (size_t)batch;
    DeviceBuffer pgb(sizeof(double) * 2 * n * B), cpb(sizeof(double) * 2 * n * B), barb(sizeof(unsigned) * 32 * B);
    DeviceBuffer aw(gmem ? sizeof(double) * B * nblk * std::max(cpc - cps, 1) * n : 0);
    PPC_CUDA_CHECK(cudaMemsetAsync(barb.d(), 0, sizeof(unsigned) * 32 * B, s));
#ifdef PPC_TRD_PROFILE
    static const bool do_prof = std::getenv("PPC_TRD_PROFILE") != nullptr;
#else
    const bool do_prof = false;
#endif
    const size_t nprof = do_prof ? (size_t)nblk * t.per_wave * (kTrdThreads / 32) * 4 : 0;
    DeviceBuffer prof(sizeof(long long) * nprof);
    if (do_prof) PPC_CUDA_CHECK(cudaMemsetAsync(prof.d(), 0, sizeof(long long) * nprof, s));
    StageTimer tm("eig.tridiag", s);
    // (1024 threads for the L2-resident variant measured no faster)
    const void* kern = (const void*)sytrd_kernel<kTrdThreads>;
    const int threads = kTrdThreads;
    PPC_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int b0 = 0; b0 < batch; b0 += t.per_wave) {
        const size_t o = (size_t)b0;
        TrdParams P;
        P.G = G + o * strideG;
        P.n = n;
        P.nblk = nblk;
        P.cpc = cpc;
        P.V = V + o * n * n;
        P.tau = tau + o * n;
        P.d = d + o * n;
        P.e = e + o * n;
        P.pg = pgb.d() + o * 2 * n;
        P.colpub = cpb.d() + o * 2 * n;
        P.bar = barb.as<unsigned>() + o * 32;
        P.Aw = gmem ? aw.d() : nullptr;
        P.cps = cps;
        P.strideG = strideG;
        P.blk = 0;
        P.prof = prof.as<long long>();
        void* args[] = {&P};
        const int nm = std::min(t.per_wave, batch - b0);
        PPC_CUDA_CHECK(cudaLaunchCooperativeKernel(kern, dim3(nblk * nm), dim3(threads),
                                                   args, smem, s));
        count_launch();
        check_launch("sytrd");
    }
    if (do_prof) {
        std::vector<long long> h(nprof);
        PPC_CUDA_CHECK(cudaMemcpyAsync(h.data(), prof.d(), sizeof(long long) * nprof, cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
        const int nw = kTrdThreads / 32;
        std::fprintf(stderr, "[trd profile] n=%d batch=%d nblk=%d cpc=%d cps=%d (last wave; kcycles per warp)\n", n, batch,
                     nblk, cpc, cps);
        for (int b = 0; b < std::min(nblk, 2); ++b)
            for (int w = 0; w < nw; w += 5) {
                const long long* q = h.data() + ((size_t)b * nw + w) * 4;
                std::fprintf(stderr, "  cta %d warp %2d: barrier %7.0f  p/w %7.0f  reflector %7.0f  update %7.0f\n", b, w,
                             q[0] * 1e-3, q[1] * 1e-3, q[2] * 1e-3, q[3] * 1e-3);
            }
    }
}

// Eigenvalues m0 .. m0 + kl - 1 (of the k wanted) of every matrix and their
// inverse-iteration vectors Z (n x kl x batch). The multisection width is
// chosen from k (not kl), so a subrange gives the same bits.
void run_vectors(const double* d, const double* e, int n, int k, int batch, int kl, int m0, double* lambda,
                 double* bnd, double* Z, cudaStream_t s) {
    {
        StageTimer tm("eig.bisect", s);
        const unsigned grid = (unsigned)(kl * batch);
        const size_t bsm = 2 * n * sizeof(double);
        if ((unsigned)(k * batch) >= 2u * (unsigned)ctx().sms)
            bisect_top_kernel<64><<<grid, 64, bsm, s>>>(d, e, n, k, lambda, bnd, kl, m0);
        else
            bisect_top_kernel<256><<<grid, 256, bsm, s>>>(d, e, n, k, lambda, bnd, kl, m0);
        count_launch();
        check_launch("bisect_top");
    }
    {
        StageTimer tm("eig.invit", s);
        const size_t ism = 7 * (size_t)n * sizeof(double) + n + 16;
        PPC_CUDA_CHECK(cudaFuncSetAttribute(inverse_iteration_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)ism));
        inverse_iteration_kernel<<<(unsigned)(kl * batch), 32, ism, s>>>(d, e, n, k, lambda, bnd, Z, kl, m0);
        count_launch();
        check_launch("inverse_iteration");
    }
}

void run_back_transform(const double* V, const double* tau, int n, int k, int batch, double* Z, cudaStream_t s) {
    StageTimer tm("eig.backtransform", s);
    DeviceBuffer Tws(sizeof(double) * ((n - 3 + kBtChunk) / kBtChunk) * kBtChunk * kBtChunk * (size_t)batch);
    if (n <= 256) launch_back_transform<8>(V, tau, n, k, batch, Z, Tws.d(), s);
    else if (n <= 512) launch_back_transform<16>(V, tau, n, k, batch, Z, Tws.d(), s);
    else if (n <= 1024) launch_back_transform<32>(V, tau, n, k, batch, Z, Tws.d(), s);
    else launch_back_transform<48>(V, tau, n, k, batch, Z, Tws.d(), s);
    count_launch();
    check_launch("back_transform");
}

}  // namespace

void tridiag_eig_top_batched(const double* G, int64_t n64, int64_t strideG, int64_t batch64, int64_t k64, double* Q,
                             double* lambda, cudaStream_t s) {
    const int n = (int)n64, k = (int)k64, batch = (int)batch64;
    if (!tridiag_eig_eligible(n64, k64, batch64)) fail(PPC_ARGUMENT, "tridiag_eig_top: size out of range");
    const size_t B = (size_t)batch;
    DeviceBuffer Vb(sizeof(double) * (size_t)n * n * B), tb(sizeof(double) * n * B), db(sizeof(double) * n * B),
        eb(sizeof(double) * n * B), bnd(sizeof(double) * 2 * B);
    run_sytrd(G, n, strideG, batch, Vb.d(), tb.d(), db.d(), eb.d(), s);
    run_vectors(db.d(), eb.d(), n, k, batch, k, 0, lambda, bnd.d(), Q, s);
    {
        StageTimer tm("eig.orth", s);
        cholqr_inplace(Q, n, k, s, batch);
    }
    run_back_transform(Vb.d(), tb.d(), n, k, batch, Q, s);
}

// ---- the eigensolve split across ranks (multi-GPU data-driven Q) ----------
EigSplit::EigSplit(const double* G, int64_t n_, int64_t p_, cudaStream_t s)
    : n(n_), p(p_), V(sizeof(double) * n_ * n_), tau(sizeof(double) * n_), d(sizeof(double) * n_),
      e(sizeof(double) * n_), lam(sizeof(double) * p_), bnd(sizeof(double) * 2) {
    run_sytrd(G, (int)n, n * n, 1, V.d(), tau.d(), d.d(), e.d(), s);
}

void EigSplit::vectors(int64_t j0, int64_t j1, double* Z, cudaStream_t s) {
    if (j0 < 0 || j1 > p || j0 >= j1) fail(PPC_BOUNDS, "eig split: eigen index range outside [0, p)");
    run_vectors(d.d(), e.d(), (int)n, (int)p, 1, (int)(j1 - j0), (int)j0, lam.d(), bnd.d(), Z, s);
}

void EigSplit::finish(double* Zall, int64_t j0, int64_t j1, double* Q, cudaStream_t s) {
    if (j0 < 0 || j1 > p || j0 >= j1) fail(PPC_BOUNDS, "eig split: column range outside [0, p)");
    {
        StageTimer tm("eig.orth", s);
        cholqr_inplace(Zall, n, p, s, 1);
    }
    PPC_CUDA_CHECK(cudaMemcpyAsync(Q, Zall + j0 * n, sizeof(double) * n * (j1 - j0), cudaMemcpyDeviceToDevice, s));
    run_back_transform(V.d(), tau.d(), (int)n, (int)(j1 - j0), 1, Q, s);
}

}  // namespace ppc
