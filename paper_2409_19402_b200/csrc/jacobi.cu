// K6 — batched one-sided (Hestenes) Jacobi SVD, one CTA per matrix.
//
// Replaces Eigen::JacobiSVD(ComputeThinU|ComputeThinV) + fix_svd_signs
// (matrix_kernels.cpp:15-37) for small slices, and serves as the small dense
// symmetric eigensolver of the engine: for a symmetric PSD H, the one-sided
// rotations that orthogonalize H's columns accumulate H's eigenvectors in V
// and the column norms of H V are its eigenvalues.
//
// Parallel round-robin ("circle") ordering: each round pairs all columns
// disjointly, one warp per pair; dot products are reduced in a fixed lane
// order (deterministic). Working set (W = R x C, V = C x C) lives in shared
// memory when it fits (<= ~200 KB), else in a global workspace (L2-resident
// for the sizes that reach this path).
#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.h"
#include "jacobi.cuh"
#include "kernels.cuh"

namespace ppc {

namespace {

constexpr double kEps = 2.220446049250313e-16;
__constant__ double c_tol_scale = 1.0;
__device__ __forceinline__ double jacobi_tol_scale() { return c_tol_scale; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Round-robin pair pi of round r among P (even) players, returned as a < c.
// 32-bit arithmetic: P <= 2^15 on every path (the working set lives in
// shared memory or an L2-resident workspace).
__device__ __forceinline__ void rr_pair(int r, int pi, int P, int& a, int& c) {
    if (pi == 0) {
        a = r;
        c = P - 1;
    } else {
        const int m = P - 1;
        a = r + pi;
        if (a >= m) a -= m;
        c = r + m - pi;
        if (c >= m) c -= m;
    }
    if (a > c) {
        const int t = a;
        a = c;
        c = t;
    }
}

// Sum over the G lanes of a lane group (fixed butterfly order, deterministic).
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One Jacobi round: every pair of the round handled by a G-lane group. Rotates the columns of W
// (R rows) and, if Va != nullptr, of Va (Cc rows); logs (cs, sn) per pair when
// lg != nullptr. Returns nonzero in *rot if any rotation was applied. Lane l
// of a group sums rows l, l+G, ... in ascending order, then a fixed butterfly.
template <int G>
__device__ __forceinline__ void jacobi_round_g(double* W, int R, double* Va, int Cc, int P, int r, double tol,
                                               double2* lg, int* rot, double gtol) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int grp = tid / G, lg_ = tid & (G - 1), ngrp = nt / G;
    const double tol2 = tol * tol;
    for (int base = 0; base < P / 2; base += ngrp) {
        const int pi = base + grp;
        // all 32 lanes of a warp stay converged for the shuffles: pairs past
        // the end work on a dummy (no memory traffic)
        const bool live = pi < P / 2;
        int a = 0, c = 0;
        if (live) rr_pair(r, pi, P, a, c);
        const bool act = live && c < Cc;
        double al = 0.0, be = 0.0, ga = 0.0;
        if (act) {
            const double* wa = W + (int64_t)a * R;
            const double* wc = W + (int64_t)c * R;
            int i = lg_;
            for (; i + 3 * G < R; i += 4 * G) {
                const double x0 = wa[i], y0 = wc[i], x1 = wa[i + G], y1 = wc[i + G];
                const double x2 = wa[i + 2 * G], y2 = wc[i + 2 * G], x3 = wa[i + 3 * G], y3 = wc[i + 3 * G];
                al = fma(x0, x0, al); be = fma(y0, y0, be); ga = fma(x0, y0, ga);
                al = fma(x1, x1, al); be = fma(y1, y1, be); ga = fma(x1, y1, ga);
                al = fma(x2, x2, al); be = fma(y2, y2, be); ga = fma(x2, y2, ga);
                al = fma(x3, x3, al); be = fma(y3, y3, be); ga = fma(x3, y3, ga);
            }
            for (; i < R; i += G) {
                const double x = wa[i], y = wc[i];
                al = fma(x, x, al);
                be = fma(y, y, be);
                ga = fma(x, y, ga);
            }
        }
        al = group_sum<G>(al);
        be = group_sum<G>(be);
        ga = group_sum<G>(ga);
        double cs = 1.0, sn = 0.0;
        // |ga| > tol sqrt(al be), compared in squares (al, be >= 0)
        if (act && ga != 0.0 && ga * ga > tol2 * (al * be) &&
            (gtol == 0.0 || fabs(ga) > gtol * (sqrt(al) + sqrt(be)))) {
            const double zeta = (be - al) / (2.0 * ga);
            const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            cs = rsqrt(1.0 + tt * tt);
            sn = cs * tt;
            double* wa = W + (int64_t)a * R;
            double* wc = W + (int64_t)c * R;
            int i = lg_;
            for (; i + G < R; i += 2 * G) {
                const double x0 = wa[i], y0 = wc[i], x1 = wa[i + G], y1 = wc[i + G];
                wa[i] = cs * x0 - sn * y0;
                wc[i] = sn * x0 + cs * y0;
                wa[i + G] = cs * x1 - sn * y1;
                wc[i + G] = sn * x1 + cs * y1;
            }
            for (; i < R; i += G) {
                const double x = wa[i], y = wc[i];
                wa[i] = cs * x - sn * y;
                wc[i] = sn * x + cs * y;
            }
            if (Va) {
                double* va = Va + (int64_t)a * Cc;
                double* vc = Va + (int64_t)c * Cc;
                int j = lg_;
                for (; j + G < Cc; j += 2 * G) {
                    const double x0 = va[j], y0 = vc[j], x1 = va[j + G], y1 = vc[j + G];
                    va[j] = cs * x0 - sn * y0;
                    vc[j] = sn * x0 + cs * y0;
                    va[j + G] = cs * x1 - sn * y1;
                    vc[j + G] = sn * x1 + cs * y1;
                }
                for (; j < Cc; j += G) {
                    const double x = va[j], y = vc[j];
                    va[j] = cs * x - sn * y;
                    vc[j] = sn * x + cs * y;
                }
            }
            if (lg_ == 0) *rot = 1;
        }
        if (lg && live && lg_ == 0) lg[pi] = make_double2(cs, sn);
    }
}

__device__ __forceinline__ void jacobi_round(double* W, int64_t R, double* Va, int64_t Cc, int64_t P, int64_t r,
                                             double tol, double2* lg, int* rot, double gtol = 0.0) {
    // 16-lane groups: measured faster than 4/8-lane groups on the 64..160
    // column eigenproblems (latency, not issue, bound with fewer warps)
    jacobi_round_g<16>(W, (int)R, Va, (int)Cc, (int)P, (int)r, tol, lg, rot, gtol);
}

__global__ void __launch_bounds__(1024, 1) jacobi_svd_kernel(const double* __restrict__ A, int64_t m, int64_t n,
                                  int64_t strideA, int64_t k, double* __restrict__ U,
                                  double* __restrict__ S, double* __restrict__ V, double* gws,
                                  int use_smem, double* tail2, int* info, double gtol_rel, int max_sweeps,
                                  const int* __restrict__ zmap) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int s_rot;
    const int64_t bz = blockIdx.x;                          // launch slot (workspace)
    const int64_t b = zmap ? (int64_t)zmap[bz] : bz;       // matrix of the batch
    const bool tall = m >= n;
    const int64_t R = tall ? m : n, Cc = tall ? n : m;
    double* W;
    double* Va;
    if (use_smem) {
        W = sm;
        Va = sm + R * Cc;
    } else {
        W = gws + bz * (R * Cc + Cc * Cc + 2 * Cc);
        Va = W + R * Cc;
    }
    double* sig = use_smem ? (Va + Cc * Cc) : (Va + Cc * Cc);
    int* rank = reinterpret_cast<int*>(sig + Cc);
    const double* Ab = A + b * strideA;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;

    // load W (= A, or A^T for wide inputs) and V = I
    for (int64_t i = tid; i < R * Cc; i += nt) {
        const int64_t r = i % R, c = i / R;
        W[i] = tall ? Ab[r + c * m] : Ab[c + r * m];
    }
    for (int64_t i = tid; i < Cc * Cc; i += nt) Va[i] = (i % Cc == i / Cc) ? 1.0 : 0.0;
    __syncthreads();

    const double tol = jacobi_tol_scale() * kEps * sqrt((double)R);
    const int64_t P = (Cc + 1) & ~int64_t(1);  // players, padded to even
    int sweep = 0;
    int* info_out = info;
    // eigenvalue-only mode: skip rotations whose effect on the Rayleigh
    // quotients is below gtol_rel * (largest column norm ~ theta_1)
    __shared__ double s_gtol;
    if (gtol_rel > 0.0) {
        if (tid == 0) s_gtol = 0.0;
        __syncthreads();
        for (int64_t c = warp; c < Cc; c += nw) {
            double acc = 0.0;
            for (int64_t i = lane; i < R; i += 32) acc = fma(W[c * R + i], W[c * R + i], acc);
            acc = warp_sum(acc);
            if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_gtol),
                                     __double_as_longlong(sqrt(acc)));
        }
        __syncthreads();
    }
    const double gtol = gtol_rel > 0.0 ? gtol_rel * s_gtol : 0.0;
    for (; sweep < max_sweeps && Cc > 1; ++sweep) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int64_t r = 0; r < P - 1; ++r) {
            jacobi_round(W, R, Va, Cc, P, r, tol, nullptr, &s_rot, gtol);
            __syncthreads();
        }
        if (!s_rot) break;
        __syncthreads();
    }

    if (tid == 0 && info_out) info_out[bz] = sweep;
    // singular values = column norms
    for (int64_t c = warp; c < Cc; c += nw) {
        double acc = 0.0;
        for (int64_t i = lane; i < R; i += 32) acc = fma(W[c * R + i], W[c * R + i], acc);
        acc = warp_sum(acc);
        if (lane == 0) sig[c] = sqrt(acc);
    }
    __syncthreads();
    // stable descending rank
    for (int64_t c = tid; c < Cc; c += nt) {
        const double sc = sig[c];
        int rk = 0;
        for (int64_t j = 0; j < Cc; ++j) {
            const double sj = sig[j];
            rk += (sj > sc) || (sj == sc && j < c);
        }
        rank[c] = rk;
    }
    __syncthreads();
    double smax = 0.0;
    for (int64_t c = 0; c < Cc; ++c) smax = fmax(smax, sig[c]);
    if (tid == 0 && tail2) {  // discarded energy, decompositions.cpp:41-49
        double acc = 0.0;
        for (int64_t c = 0; c < Cc; ++c)
            if (rank[c] >= k) acc = fma(sig[c], sig[c], acc);
        tail2[b] = acc;
    }
    const double ztol = smax * kEps * (double)R;

    // outputs: the wide case swaps roles (A^T = U' S V'^T => A = V' S U'^T)
    double* Uo = U ? U + b * m * k : nullptr;
    double* Vo = V ? V + b * n * k : nullptr;
    double* Ltall = tall ? Uo : Vo;  // receives normalized W columns (R rows)
    double* Lrot = tall ? Vo : Uo;   // receives rotation columns (Cc rows)
    for (int64_t c = warp; c < Cc; c += nw) {
        const int64_t o = rank[c];
        if (o >= k) continue;
        const double s = sig[c];
        if (lane == 0 && S) S[b * k + o] = s;
        if (Ltall) {
            const double inv = (s > ztol && s > 0.0) ? 1.0 / s : 0.0;
            for (int64_t i = lane; i < R; i += 32) Ltall[o * R + i] = W[c * R + i] * inv;
        }
        if (Lrot)
            for (int64_t i = lane; i < Cc; i += 32) Lrot[o * Cc + i] = Va[c * Cc + i];
    }
    __syncthreads();
    if (!U) return;  // eigen mode: no left vectors, no sign rule needed by callers
    // orthonormal completion of zero-sigma columns of the tall factor
    // (JacobiSVD's thin U is always orthonormal), warp 0, in column order
    if (Ltall && warp == 0) {
        for (int64_t o = 0; o < k && o < Cc; ++o) {
            // find sigma of output column o
            double so = 0.0;
            for (int64_t c = 0; c < Cc; ++c)
                if (rank[c] == o) so = sig[c];
            if (so > ztol && so > 0.0) continue;
            double* col = Ltall + o * R;
            for (int64_t e = 0; e < R; ++e) {
                for (int64_t i = lane; i < R; i += 32) col[i] = (i == e) ? 1.0 : 0.0;
                __syncwarp();
                for (int pass = 0; pass < 2; ++pass)
                    for (int64_t q = 0; q < k && q < Cc; ++q) {
                        if (q == o) continue;
                        double sq = 0.0;
                        for (int64_t c = 0; c < Cc; ++c)
                            if (rank[c] == q) sq = sig[c];
                        if (q > o && !(sq > ztol && sq > 0.0)) continue;  // not yet filled
                        const double* u = Ltall + q * R;
                        double d = 0.0;
                        for (int64_t i = lane; i < R; i += 32) d = fma(u[i], col[i], d);
                        d = warp_sum(d);
                        for (int64_t i = lane; i < R; i += 32) col[i] -= d * u[i];
                        __syncwarp();
                    }
                double nv = 0.0;
                for (int64_t i = lane; i < R; i += 32) nv = fma(col[i], col[i], nv);
                nv = sqrt(warp_sum(nv));
                if (nv > 0.5) {
                    for (int64_t i = lane; i < R; i += 32) col[i] /= nv;
                    __syncwarp();
                    break;
                }
            }
        }
    }
    __syncthreads();
    // sign rule (matrix_kernels.cpp:16-25): largest |U| entry (first on ties)
    // of each U column made nonnegative, V flipped with it.
    for (int64_t o = warp; o < k && o < Cc; o += nw) {
        const double* u = Uo + o * m;
        double best = -1.0;
        int64_t bi = 0;
        for (int64_t i = lane; i < m; i += 32) {
            const double a = fabs(u[i]);
            if (a > best) { best = a; bi = i; }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        const bool flip = u[bi] < 0.0;
        __syncwarp();
        if (flip) {
            for (int64_t i = lane; i < m; i += 32) Uo[o * m + i] = -Uo[o * m + i];
            if (Vo)
                for (int64_t i = lane; i < n; i += 32) Vo[o * n + i] = -Vo[o * n + i];
        }
    }
}


// Eigen mode for symmetric PSD blocks whose W fits shared memory but W + V do
// not (b <= ~160): sweep on W in shared memory and log every round's
// rotations (cs, sn) to global memory; V is rebuilt afterwards by a
// row-parallel kernel that replays the log. rank/sig go to global memory.
__global__ void __launch_bounds__(1024, 1) jacobi_logged_kernel(const double* __restrict__ A, int64_t b, int64_t strideA,
                                     double2* __restrict__ log, int64_t max_sweeps,
                                     int* __restrict__ nsweeps, double* __restrict__ sig_out,
                                     int* __restrict__ rank_out, double gtol_rel,
                                     const int* __restrict__ zmap) {
    extern __shared__ __align__(16) double W[];
    __shared__ int s_rot;
    const int64_t bi = blockIdx.x;  // launch slot: log / sweeps / sig / rank
    const double* Ab = A + (zmap ? (int64_t)zmap[bi] : bi) * strideA;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
    for (int64_t i = tid; i < b * b; i += nt) W[i] = Ab[i];
    __syncthreads();
    const int64_t P = (b + 1) & ~int64_t(1);
    const int64_t per_sweep = (P - 1) * (P / 2);
    double2* lg = log + bi * max_sweeps * per_sweep;
    const double tol = jacobi_tol_scale() * kEps * sqrt((double)b);
    int sweep = 0;
    __shared__ double s_gtol;
    if (gtol_rel > 0.0) {
        if (tid == 0) s_gtol = 0.0;
        __syncthreads();
        for (int64_t c = warp; c < b; c += nw) {
            double acc = 0.0;
            for (int64_t i = lane; i < b; i += 32) acc = fma(W[c * b + i], W[c * b + i], acc);
            acc = warp_sum(acc);
            if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_gtol),
                                     __double_as_longlong(sqrt(acc)));
        }
        __syncthreads();
    }
    const double gtol = gtol_rel > 0.0 ? gtol_rel * s_gtol : 0.0;
    for (; sweep < max_sweeps && b > 1; ++sweep) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int64_t r = 0; r < P - 1; ++r) {
            jacobi_round(W, b, nullptr, b, P, r, tol, lg + sweep * per_sweep + r * (P / 2), &s_rot, gtol);
            __syncthreads();
        }
        if (!s_rot) { ++sweep; break; }
        __syncthreads();
    }
    if (tid == 0) nsweeps[bi] = sweep;
    double* sig = sig_out + bi * b;
    int* rank = rank_out + bi * b;
    for (int64_t c = warp; c < b; c += nw) {
        double acc = 0.0;
        for (int64_t i = lane; i < b; i += 32) acc = fma(W[c * b + i], W[c * b + i], acc);
        acc = warp_sum(acc);
        if (lane == 0) sig[c] = sqrt(acc);
    }
    __syncthreads();
    for (int64_t c = tid; c < b; c += nt) {
        const double sc = sig[c];
        int rk = 0;
        for (int64_t j = 0; j < b; ++j) rk += (sig[j] > sc) || (sig[j] == sc && j < c);
        rank[c] = rk;
    }
}

// Replays the rotation log on rows [row0, row0+ROWS) of V = I, then writes
// the leading k eigenvectors (columns in rank order) and eigenvalues.
template <int ROWS>
__global__ void replay_rotations_kernel(const double2* __restrict__ log, const int* __restrict__ nsweeps,
                                        int64_t b, int64_t max_sweeps, const double* __restrict__ sig,
                                        const int* __restrict__ rank, int64_t k, double* __restrict__ V,
                                        double* __restrict__ lambda, const int* __restrict__ zmap) {
    extern __shared__ __align__(16) double Vr[];  // ROWS x b, row-major
    const int64_t bi = blockIdx.y;
    const int64_t row0 = (int64_t)blockIdx.x * ROWS;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int64_t t = tid; t < ROWS * b; t += nt) {
        const int64_t i = t / b, c = t % b;
        Vr[t] = (row0 + i == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    const int64_t P = (b + 1) & ~int64_t(1);
    const int64_t per_sweep = (P - 1) * (P / 2);
    const double2* lg = log + bi * max_sweeps * per_sweep;
    const int sw = nsweeps[bi];
    for (int s = 0; s < sw; ++s)
        for (int64_t r = 0; r < P - 1; ++r) {
            const double2* rl = lg + s * per_sweep + r * (P / 2);
            for (int64_t t = tid; t < ROWS * (P / 2); t += nt) {
                const int64_t i = t / (P / 2), pi = t % (P / 2);
                const double2 cs = rl[pi];
                if (cs.y == 0.0 && cs.x == 1.0) continue;
                int64_t a, c;
                if (pi == 0) { a = r; c = P - 1; }
                else { a = (r + pi) % (P - 1); c = (r + P - 1 - pi) % (P - 1); }
                if (a > c) { int64_t tq = a; a = c; c = tq; }
                if (c >= b) continue;
                double* v = Vr + i * b;
                const double x = v[a], y = v[c];
                v[a] = cs.x * x - cs.y * y;
                v[c] = cs.y * x + cs.x * y;
            }
            __syncthreads();
        }
    const int* rk = rank + bi * b;
    const int64_t bo = zmap ? (int64_t)zmap[bi] : bi;  // output matrix of the batch
    for (int64_t t = tid; t < ROWS * b; t += nt) {
        const int64_t i = t / b, c = t % b;
        const int64_t o = rk[c];
        if (o < k && row0 + i < b) V[(bo * k + o) * b + row0 + i] = Vr[t];
    }
    if (blockIdx.x == 0)
        for (int64_t c = tid; c < b; c += nt)
            if (rk[c] < k) lambda[bo * k + rk[c]] = sig[bi * b + c];
}

}  // namespace

size_t jacobi_smem_bytes(int64_t m, int64_t n) {
    const int64_t R = m > n ? m : n, C = m > n ? n : m;
    return (size_t)(R * C + C * C + C) * sizeof(double) + (size_t)C * sizeof(int) + 16;
}

void jacobi_svd(const double* A, int64_t m, int64_t n, int64_t strideA, int64_t batch, int64_t k,
                double* U, double* S, double* V, double* tail2, cudaStream_t s, double gtol_rel,
                int sweep_cap, const int* zmap) {
    HostProf hp_("jacobi_svd");
    if (batch == 0) return;
    static std::atomic<uint64_t> tol_set{0};  // the symbol lives in each device's module
    once_per_device(tol_set, [] {
        const char* e = std::getenv("PPC_JACOBI_TOL");
        const double v = e ? std::atof(e) : 1.0;
        PPC_CUDA_CHECK(cudaMemcpyToSymbol(c_tol_scale, &v, sizeof(double)));
    });
    const int64_t R = m > n ? m : n, C = m > n ? n : m;
    if (k < 1 || k > C) fail(PPC_ARGUMENT, "jacobi_svd: k out of range");
    const size_t smem = jacobi_smem_bytes(m, n);
    const int threads = C >= 96 ? 1024 : (C >= 48 ? 512 : (C >= 24 ? 256 : 128));
    const bool use_smem = smem <= 200 * 1024;
    if (!use_smem && !U && !tail2 && m == n && (size_t)n * n * sizeof(double) <= 200 * 1024) {
        // eigen mode, W fits but W + V does not: logged rotations + replay
        const int64_t P = (n + 1) & ~int64_t(1);
        const int64_t max_sweeps = sweep_cap > 0 ? std::min(sweep_cap, 40) : 40;
        DeviceBuffer lg(sizeof(double2) * batch * max_sweeps * (P - 1) * (P / 2)),
            ns(sizeof(int) * batch), sg(sizeof(double) * batch * n), rk(sizeof(int) * batch * n);
        const size_t wsm = (size_t)n * n * sizeof(double);
        PPC_CUDA_CHECK(cudaFuncSetAttribute(jacobi_logged_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
        jacobi_logged_kernel<<<(unsigned)batch, 1024, wsm, s>>>(A, n, strideA, lg.as<double2>(),
                                                                max_sweeps, ns.as<int>(), sg.d(),
                                                                rk.as<int>(), gtol_rel, zmap);
        count_launch();
        check_launch("jacobi_logged");
        constexpr int ROWS = 8;
        const size_t rsm = (size_t)ROWS * n * sizeof(double);
        PPC_CUDA_CHECK(cudaFuncSetAttribute(replay_rotations_kernel<ROWS>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
        dim3 grid((unsigned)((n + ROWS - 1) / ROWS), (unsigned)batch);
        replay_rotations_kernel<ROWS><<<grid, 256, rsm, s>>>(lg.as<double2>(), ns.as<int>(), n,
                                                             max_sweeps, sg.d(), rk.as<int>(), k,
                                                             V, S, zmap);
        count_launch();
        check_launch("replay_rotations");
        if (std::getenv("PPC_JACOBI_DEBUG")) {
            std::vector<int> h(batch);
            PPC_CUDA_CHECK(cudaMemcpyAsync(h.data(), ns.d(), sizeof(int) * batch, cudaMemcpyDeviceToHost, s));
            PPC_CUDA_CHECK(cudaStreamSynchronize(s));
            fprintf(stderr, "[jacobi-logged] %lldx%lld batch %lld sweeps %d\n", (long long)n, (long long)n,
                    (long long)batch, h[0]);
        }
        return;
    }
    DeviceBuffer ws;
    if (!use_smem) ws = DeviceBuffer((size_t)batch * (R * C + C * C + 2 * C) * sizeof(double));
    if (use_smem && smem > 48 * 1024)
        PPC_CUDA_CHECK(cudaFuncSetAttribute(jacobi_svd_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (batch > 0x7fffffffLL) fail(PPC_ARGUMENT, "jacobi_svd: batch too large");
    static const bool dbg = std::getenv("PPC_JACOBI_DEBUG") != nullptr;
    DeviceBuffer dinfo(sizeof(int) * batch);
    jacobi_svd_kernel<<<(unsigned)batch, threads, use_smem ? smem : 0, s>>>(
        A, m, n, strideA, k, U, S, V, ws.d(), use_smem ? 1 : 0, tail2, dinfo.as<int>(), gtol_rel,
        sweep_cap > 0 ? sweep_cap : 60, zmap);
    count_launch();
    check_launch("jacobi_svd");
    if (dbg) {
        std::vector<int> h(batch);
        PPC_CUDA_CHECK(cudaMemcpyAsync(h.data(), dinfo.d(), sizeof(int) * batch, cudaMemcpyDeviceToHost, s));
        PPC_CUDA_CHECK(cudaStreamSynchronize(s));
        int mx = 0;
        long sum = 0;
        for (int v : h) { mx = std::max(mx, v); sum += v; }
        fprintf(stderr, "[jacobi] %lldx%lld batch %lld k %lld smem %d sweeps max %d avg %.1f\n", (long long)m,
                (long long)n, (long long)batch, (long long)k, use_smem ? 1 : 0, mx, (double)sum / batch);
    }
}

}  // namespace ppc

namespace ppc {
namespace {
__global__ void sign_rule_kernel(double* X, int64_t rows, int64_t cols, double* Y, int64_t yrows) {
    const int64_t b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (c >= cols) return;
    double* x = X + (b * cols + c) * rows;
    double best = -1.0;
    int64_t bi = 0;
    for (int64_t i = lane; i < rows; i += 32) {
        const double a = fabs(x[i]);
        if (a > best) { best = a; bi = i; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, off);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const bool flip = x[bi] < 0.0;
    __syncwarp();
    if (!flip) return;
    for (int64_t i = lane; i < rows; i += 32) x[i] = -x[i];
    if (Y) {
        double* y = Y + (b * cols + c) * yrows;
        for (int64_t i = lane; i < yrows; i += 32) y[i] = -y[i];
    }
}
}  // namespace

void sign_rule(double* X, int64_t rows, int64_t cols, int64_t batch, double* Y, int64_t yrows,
               cudaStream_t s) {
    if (!cols || !batch) return;
    dim3 grid((unsigned)((cols + 7) / 8), (unsigned)batch);
    sign_rule_kernel<<<grid, 256, 0, s>>>(X, rows, cols, Y, yrows);
    count_launch();
    check_launch("sign_rule");
}
}  // namespace ppc
