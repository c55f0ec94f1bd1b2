/*
 * ppo.c — CPU oracle (TEST INFRASTRUCTURE ONLY; see ppo.h).
 *
 * Plain-C restatement of the reference hot path. Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Eigen (the reference's arithmetic library, not vendored, unpinned:
 * proj/CMakeLists.txt:15 "find_package(Eigen3 3.3 REQUIRED)") is replaced by:
 *   - GEMM: a blocked column-major triple loop (or an optional OpenBLAS dgemm
 *     via ppo_use_blas for the CPU baseline);
 *   - Eigen::JacobiSVD: one-sided (Hestenes) cyclic Jacobi, converged to
 *     machine precision, descending sort, then the reference sign rule;
 *   - Eigen::HouseholderQR: textbook Householder QR.
 * Parity with the reference is by contract (tolerances in the reference's own
 * tests), which is how the reference's tests pin Eigen as well.
 */
#define _GNU_SOURCE
#include "ppo.h"

#include <dlfcn.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------ errors */
static __thread char g_err[512];
const char* ppo_last_error(void) { return g_err; }
static int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
#include <stdarg.h>
static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* --------------------------------------------------------------- threading */
/* parallel.cpp:13-27: min(hardware, PROJPROD_THREADS), <1 clamps to 1. */
static int g_threads = 0;
void ppo_set_threads(int n) { g_threads = n; }
int ppo_threads(void) {
    if (g_threads > 0) return g_threads;
    long hw = sysconf(_SC_NPROCESSORS_ONLN);
    if (hw < 1) hw = 1;
    const char* env = getenv("PROJPROD_THREADS");
    if (env && *env) {
        char* end = NULL;
        long cap = strtol(env, &end, 10);
        if (end != env) {
            if (cap < 1) cap = 1;
            if (cap < hw) hw = cap;
        }
    }
    return (int)hw;
}

typedef void (*body_fn)(int64_t i, void* ctx);
typedef struct { int64_t lo, hi; body_fn fn; void* ctx; } chunk_t;
static void* run_chunk(void* arg) {
    chunk_t* c = (chunk_t*)arg;
    for (int64_t i = c->lo; i < c->hi; ++i) c->fn(i, c->ctx);
    return NULL;
}
/* parallel.cpp:29-57: contiguous chunks over at most max_threads workers. */
static void parallel_for(int64_t n, body_fn fn, void* ctx) {
    if (n <= 0) return;
    int64_t workers = ppo_threads();
    if (workers > n) workers = n;
    if (workers <= 1) {
        for (int64_t i = 0; i < n; ++i) fn(i, ctx);
        return;
    }
    pthread_t th[256];
    chunk_t ch[256];
    if (workers > 256) workers = 256;
    int64_t chunk = (n + workers - 1) / workers;
    int started = 0;
    for (int64_t w = 0; w < workers; ++w) {
        int64_t lo = w * chunk, hi = lo + chunk < n ? lo + chunk : n;
        if (lo >= hi) break;
        ch[w] = (chunk_t){lo, hi, fn, ctx};
        pthread_create(&th[w], NULL, run_chunk, &ch[w]);
        started++;
    }
    for (int w = 0; w < started; ++w) pthread_join(th[w], NULL);
}

/* -------------------------------------------------------------------- GEMM */
typedef void (*dgemm_t)(const char*, const char*, const int*, const int*, const int*,
                        const double*, const double*, const int*, const double*,
                        const int*, const double*, double*, const int*);
static dgemm_t g_dgemm = NULL;
static void (*g_blas_threads)(int) = NULL;

int ppo_use_blas(const char* path, const char* sym, const char* set_threads_sym) {
    void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) return fail(PPO_ARGUMENT, "dlopen %s failed: %s", path, dlerror());
    g_dgemm = (dgemm_t)dlsym(h, sym);
    if (!g_dgemm) return fail(PPO_ARGUMENT, "symbol %s not found", sym);
    if (set_threads_sym && *set_threads_sym) {
        g_blas_threads = (void (*)(int))dlsym(h, set_threads_sym);
        if (g_blas_threads) g_blas_threads(1); /* Eigen without OpenMP: single-threaded GEMM (CMakeLists.txt:30) */
    }
    return 0;
}

/* Threads of the BLAS GEMMs (1 by default, as the reference). The parity
 * tests raise it to check BASELINE-sized products in seconds; the CPU
 * baseline keeps the reference's single thread per GEMM. */
int ppo_set_blas_threads(int n) {
    if (!g_dgemm || !g_blas_threads) return fail(PPO_ARGUMENT, "no BLAS loaded");
    g_blas_threads(n < 1 ? 1 : n);
    return 0;
}

/* C(m x n) = alpha * op(A) * op(B) + beta * C, column-major, op in {N,T}. */
static void gemm(char ta, char tb, int64_t m, int64_t n, int64_t k, double alpha,
                 const double* A, int64_t lda, const double* B, int64_t ldb,
                 double beta, double* C, int64_t ldc) {
    if (m <= 0 || n <= 0) return;
    if (g_dgemm && m < 2147483647 && n < 2147483647 && k < 2147483647 && k > 0) {
        int M = (int)m, N = (int)n, K = (int)k, LA = (int)lda, LB = (int)ldb, LC = (int)ldc;
        g_dgemm(&ta, &tb, &M, &N, &K, &alpha, A, &LA, B, &LB, &beta, C, &LC);
        return;
    }
    for (int64_t j = 0; j < n; ++j) {
        double* c = C + j * ldc;
        if (beta == 0.0)
            for (int64_t i = 0; i < m; ++i) c[i] = 0.0;
        else if (beta != 1.0)
            for (int64_t i = 0; i < m; ++i) c[i] *= beta;
    }
    if (k <= 0) return;
    const int64_t MB = 512, KB = 128;
    if (ta == 'N') {
        for (int64_t i0 = 0; i0 < m; i0 += MB) {
            int64_t mb = m - i0 < MB ? m - i0 : MB;
            for (int64_t p0 = 0; p0 < k; p0 += KB) {
                int64_t kb = k - p0 < KB ? k - p0 : KB;
                for (int64_t j = 0; j < n; ++j) {
                    double* c = C + j * ldc + i0;
                    for (int64_t p = p0; p < p0 + kb; ++p) {
                        double b = (tb == 'N') ? B[p + j * ldb] : B[j + p * ldb];
                        if (b == 0.0) continue;
                        b *= alpha;
                        const double* a = A + p * lda + i0;
                        for (int64_t i = 0; i < mb; ++i) c[i] += a[i] * b;
                    }
                }
            }
        }
    } else { /* A^T: dot products over contiguous columns of A */
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < m; ++i) {
                const double* a = A + i * lda;
                double acc = 0.0;
                if (tb == 'N') {
                    const double* b = B + j * ldb;
                    for (int64_t p = 0; p < k; ++p) acc += a[p] * b[p];
                } else {
                    for (int64_t p = 0; p < k; ++p) acc += a[p] * B[j + p * ldb];
                }
                C[i + j * ldc] += alpha * acc;
            }
    }
}

/* ----------------------------------------------------------------- RNG */
/* rng.hpp:12-18 */
static uint64_t splitmix64(uint64_t* x) {
    *x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
/* rng.hpp:21-26 */
uint64_t ppo_derive_seed(uint64_t seed, uint64_t stream) {
    uint64_t x = seed ^ (0xa0761d6478bd642fULL * (stream + 1));
    uint64_t a = splitmix64(&x);
    uint64_t b = splitmix64(&x);
    return a ^ (b << 1);
}
typedef struct { uint64_t s[4]; double spare; int has_spare; } xoshiro_t;
static uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
static void xo_init(xoshiro_t* r, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&x);
    r->has_spare = 0;
    r->spare = 0.0;
}
/* rng.hpp:36-47 */
static uint64_t xo_next(xoshiro_t* r) {
    uint64_t* s = r->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}
static double xo_uniform(xoshiro_t* r) { return (double)(xo_next(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:56-69 Box-Muller with cached spare */
static double xo_normal(xoshiro_t* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = xo_uniform(r), u2 = xo_uniform(r);
    while (u1 <= 0.0) u1 = xo_uniform(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    r->spare = rad * sin(theta);
    r->has_spare = 1;
    return rad * cos(theta);
}
void ppo_xoshiro_normals(uint64_t seed, double* out, int64_t count) {
    xoshiro_t r;
    xo_init(&r, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = xo_normal(&r);
}

/* ------------------------------------------------------------ tensor core */
double ppo_frobenius_norm(const double* A, int64_t count) {
    /* plain sum of squares; tensor.cpp:158 uses Eigen's norm() */
    double acc = 0.0;
    for (int64_t i = 0; i < count; ++i) acc += A[i] * A[i];
    return sqrt(acc);
}

int ppo_mode3_product(const double* A, int64_t n1, int64_t n2, int64_t n3,
                      const double* M, int64_t q, double* out) {
    if (n1 < 1 || n2 < 1 || n3 < 1 || q < 1)
        return fail(PPO_SHAPE, "mode3_product: extents must be positive");
    const int64_t N = n1 * n2;
    /* out.tubes (N x q) = A.tubes (N x n3) * M^T (n3 x q); M is q x n3. */
    gemm('N', 'T', N, q, n3, 1.0, A, N, M, q, 0.0, out, N);
    return 0;
}

typedef struct {
    const double *A, *B;
    double* C;
    int64_t n1, m, n2;
} face_ctx;
static void face_body(int64_t s, void* vctx) {
    face_ctx* c = (face_ctx*)vctx;
    gemm('N', 'N', c->n1, c->n2, c->m, 1.0, c->A + s * c->n1 * c->m, c->n1,
         c->B + s * c->m * c->n2, c->m, 0.0, c->C + s * c->n1 * c->n2, c->n1);
}
int ppo_facewise_product(const double* A, int64_t n1, int64_t m, int64_t n3,
                         const double* B, int64_t n2, double* C) {
    if (n1 < 1 || m < 1 || n3 < 1 || n2 < 1)
        return fail(PPO_SHAPE, "facewise_product: extents must be positive");
    face_ctx c = {A, B, C, n1, m, n2};
    parallel_for(n3, face_body, &c);
    return 0;
}

/* ------------------------------------------------------- one-sided Jacobi */
/* Hestenes one-sided Jacobi on W (m x n, m >= n), accumulating V (n x n).
 * On exit column norms of W are the singular values (unsorted). */
static void hestenes(double* W, int64_t m, int64_t n, double* V) {
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) V[i + j * n] = (i == j) ? 1.0 : 0.0;
    const double tol = 2.220446049250313e-16;
    for (int sweep = 0; sweep < 80; ++sweep) {
        int rotated = 0;
        for (int64_t i = 0; i < n - 1; ++i) {
            double* wi = W + i * m;
            for (int64_t j = i + 1; j < n; ++j) {
                double* wj = W + j * m;
                double a = 0, b = 0, g = 0;
                for (int64_t r = 0; r < m; ++r) {
                    a += wi[r] * wi[r];
                    b += wj[r] * wj[r];
                    g += wi[r] * wj[r];
                }
                if (g == 0.0 || fabs(g) <= tol * sqrt(a * b)) continue;
                rotated = 1;
                const double zeta = (b - a) / (2.0 * g);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (int64_t r = 0; r < m; ++r) {
                    const double x = wi[r], y = wj[r];
                    wi[r] = c * x - s * y;
                    wj[r] = s * x + c * y;
                }
                double* vi = V + i * n;
                double* vj = V + j * n;
                for (int64_t r = 0; r < n; ++r) {
                    const double x = vi[r], y = vj[r];
                    vi[r] = c * x - s * y;
                    vj[r] = s * x + c * y;
                }
            }
        }
        if (!rotated) break;
    }
}

/* Fill zero columns of U (m x r) with an orthonormal completion (Gram-Schmidt
 * of canonical vectors, twice). Eigen's thin U is always orthonormal. */
static void complete_columns(double* U, int64_t m, int64_t r, const int* zero) {
    double* v = (double*)malloc(sizeof(double) * m);
    int64_t e = 0;
    for (int64_t j = 0; j < r; ++j) {
        if (!zero[j]) continue;
        for (; e < m; ++e) {
            for (int64_t i = 0; i < m; ++i) v[i] = (i == e) ? 1.0 : 0.0;
            for (int pass = 0; pass < 2; ++pass)
                for (int64_t c = 0; c < r; ++c) {
                    if (c == j || (zero[c] && c > j)) continue;
                    const double* u = U + c * m;
                    double d = 0;
                    for (int64_t i = 0; i < m; ++i) d += u[i] * v[i];
                    for (int64_t i = 0; i < m; ++i) v[i] -= d * u[i];
                }
            double nv = 0;
            for (int64_t i = 0; i < m; ++i) nv += v[i] * v[i];
            nv = sqrt(nv);
            if (nv > 0.5) {
                for (int64_t i = 0; i < m; ++i) U[i + j * m] = v[i] / nv;
                ++e;
                break;
            }
        }
    }
    free(v);
}

/* matrix_kernels.cpp:16-25: largest-|U| entry (first on ties) >= 0; V follows. */
static void fix_svd_signs(double* U, int64_t m, double* V, int64_t n, int64_t r) {
    for (int64_t j = 0; j < r; ++j) {
        int64_t imax = 0;
        double best = -1.0;
        for (int64_t i = 0; i < m; ++i) {
            double a = fabs(U[i + j * m]);
            if (a > best) { best = a; imax = i; }
        }
        if (U[imax + j * m] < 0.0) {
            for (int64_t i = 0; i < m; ++i) U[i + j * m] = -U[i + j * m];
            for (int64_t i = 0; i < n; ++i) V[i + j * n] = -V[i + j * n];
        }
    }
}

/* Thin SVD of a tall W (m x n, m >= n) into U (m x n), s (n), V (n x n). */
static void svd_tall(const double* A, int64_t m, int64_t n, double* U, double* s, double* V) {
    double* W = (double*)malloc(sizeof(double) * m * n);
    double* Vt = (double*)malloc(sizeof(double) * n * n);
    memcpy(W, A, sizeof(double) * m * n);
    hestenes(W, m, n, Vt);
    double* sig = (double*)malloc(sizeof(double) * n);
    int64_t* ord = (int64_t*)malloc(sizeof(int64_t) * n);
    int* zero = (int*)calloc((size_t)n, sizeof(int));
    double smax = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        double acc = 0;
        for (int64_t i = 0; i < m; ++i) acc += W[i + j * m] * W[i + j * m];
        sig[j] = sqrt(acc);
        if (sig[j] > smax) smax = sig[j];
        ord[j] = j;
    }
    /* stable insertion sort, descending */
    for (int64_t a = 1; a < n; ++a) {
        int64_t x = ord[a];
        int64_t b = a - 1;
        while (b >= 0 && sig[ord[b]] < sig[x]) { ord[b + 1] = ord[b]; --b; }
        ord[b + 1] = x;
    }
    const double ztol = smax * 2.220446049250313e-16 * (double)(m > n ? m : n);
    for (int64_t c = 0; c < n; ++c) {
        int64_t j = ord[c];
        s[c] = sig[j];
        if (sig[j] <= ztol || sig[j] == 0.0) {
            zero[c] = 1;
            for (int64_t i = 0; i < m; ++i) U[i + c * m] = 0.0;
        } else {
            for (int64_t i = 0; i < m; ++i) U[i + c * m] = W[i + j * m] / sig[j];
        }
        for (int64_t i = 0; i < n; ++i) V[i + c * n] = Vt[i + j * n];
    }
    complete_columns(U, m, n, zero);
    free(W); free(Vt); free(sig); free(ord); free(zero);
}

static int all_finite(const double* A, int64_t count) {
    for (int64_t i = 0; i < count; ++i)
        if (!isfinite(A[i])) return 0;
    return 1;
}

/* matrix_kernels.cpp:29-37 */
int ppo_svd(const double* A, int64_t m, int64_t n, double* U, double* s, double* V) {
    if (m < 1 || n < 1) return fail(PPO_SHAPE, "svd: empty matrix");
    if (!all_finite(A, m * n)) return fail(PPO_NUMERIC, "svd: input has non-finite entries");
    const int64_t r = m < n ? m : n;
    if (m >= n) {
        svd_tall(A, m, n, U, s, V);
    } else {
        /* A^T (n x m) = U' S V'^T  =>  A = V' S U'^T */
        double* At = (double*)malloc(sizeof(double) * m * n);
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < m; ++i) At[j + i * n] = A[i + j * m];
        svd_tall(At, n, m, V, s, U); /* V: n x m, U: m x m */
        free(At);
    }
    fix_svd_signs(U, m, V, n, r);
    return 0;
}

/* ------------------------------------------------------------ Householder */
/* In-place Householder QR of A (m x n, m >= n); tau[n]; R in the upper
 * triangle, reflectors below (LAPACK dgeqrf convention). */
static void householder_qr(double* A, int64_t m, int64_t n, double* tau) {
    for (int64_t j = 0; j < n; ++j) {
        double* a = A + j * m;
        double nrm = 0;
        for (int64_t i = j + 1; i < m; ++i) nrm += a[i] * a[i];
        const double alpha = a[j];
        if (nrm == 0.0) { tau[j] = 0.0; continue; }
        double beta = -copysign(sqrt(alpha * alpha + nrm), alpha);
        tau[j] = (beta - alpha) / beta;
        const double scale = 1.0 / (alpha - beta);
        for (int64_t i = j + 1; i < m; ++i) a[i] *= scale;
        a[j] = beta;
        /* apply H = I - tau v v^T (v = [1; a[j+1:]]) to the trailing columns */
        for (int64_t c = j + 1; c < n; ++c) {
            double* b = A + c * m;
            double d = b[j];
            for (int64_t i = j + 1; i < m; ++i) d += a[i] * b[i];
            d *= tau[j];
            b[j] -= d;
            for (int64_t i = j + 1; i < m; ++i) b[i] -= d * a[i];
        }
    }
}
/* Q(:,0:p) = H_0 ... H_{n-1} I(:,0:p) */
static void householder_form_q(const double* QR, int64_t m, int64_t n, const double* tau,
                               int64_t p, double* Q) {
    for (int64_t j = 0; j < p; ++j)
        for (int64_t i = 0; i < m; ++i) Q[i + j * m] = (i == j) ? 1.0 : 0.0;
    for (int64_t j = n - 1; j >= 0; --j) {
        const double* v = QR + j * m;
        if (tau[j] == 0.0) continue;
        for (int64_t c = 0; c < p; ++c) {
            double* b = Q + c * m;
            double d = b[j];
            for (int64_t i = j + 1; i < m; ++i) d += v[i] * b[i];
            d *= tau[j];
            b[j] -= d;
            for (int64_t i = j + 1; i < m; ++i) b[i] -= d * v[i];
        }
    }
}

/* matrix_kernels.cpp:93-101 */
static int64_t numerical_rank(const double* s, int64_t r, double tol_rel) {
    if (r == 0) return 0;
    const double cutoff = tol_rel * s[0];
    int64_t k = 0;
    while (k < r && s[k] > cutoff) ++k;
    return k;
}

/* matrix_kernels.cpp:48-78 */
int ppo_orthonormalize(const double* A, int64_t n, int64_t p, double* Q) {
    if (p < 1 || p > n) return fail(PPO_ARGUMENT, "orthonormalize: need 1 <= cols <= rows, got %ldx%ld", (long)n, (long)p);
    if (!all_finite(A, n * p)) return fail(PPO_NUMERIC, "orthonormalize: input has non-finite entries");
    double* U = (double*)malloc(sizeof(double) * n * p);
    double* s = (double*)malloc(sizeof(double) * p);
    double* V = (double*)malloc(sizeof(double) * p * p);
    ppo_svd(A, n, p, U, s, V);
    int64_t rank = numerical_rank(s, p, 1e-12);
    free(U); free(V); free(s);
    if (rank < p) return fail(PPO_DEGENERATE, "orthonormalize: input is rank-deficient (rank %ld < %ld)", (long)rank, (long)p);
    double* QR = (double*)malloc(sizeof(double) * n * p);
    double* tau = (double*)malloc(sizeof(double) * p);
    memcpy(QR, A, sizeof(double) * n * p);
    householder_qr(QR, n, p, tau);
    householder_form_q(QR, n, p, tau, p, Q);
    free(QR); free(tau);
    for (int64_t j = 0; j < p; ++j)
        for (int64_t i = 0; i < n; ++i) {
            if (fabs(Q[i + j * n]) > 1e-12) {
                if (Q[i + j * n] < 0.0)
                    for (int64_t r = 0; r < n; ++r) Q[r + j * n] = -Q[r + j * n];
                break;
            }
        }
    return 0;
}

/* ------------------------------------------------------------- transforms */
static int check_dims(int64_t n3, int64_t p) {
    if (n3 < 1) return fail(PPO_ARGUMENT, "transform: n3 must be positive");
    if (p < 1 || p > n3) return fail(PPO_ARGUMENT, "transform: p=%ld outside [1,%ld]", (long)p, (long)n3);
    return 0;
}

int ppo_dct_q(int64_t n3, int64_t p, double* Q) {
    int rc = check_dims(n3, p);
    if (rc) return rc;
    const double n = (double)n3;
    for (int64_t j = 0; j < p; ++j) {
        const double w = (j == 0) ? sqrt(1.0 / n) : sqrt(2.0 / n);
        for (int64_t t = 0; t < n3; ++t)
            Q[t + j * n3] = w * cos(3.14159265358979323846 * (2.0 * t + 1.0) * j / (2.0 * n));
    }
    return 0;
}

int ppo_random_orthogonal_q(int64_t n3, int64_t p, uint64_t seed, double* Q) {
    int rc = check_dims(n3, p);
    if (rc) return rc;
    double* G = (double*)malloc(sizeof(double) * n3 * n3);
    double* F = (double*)malloc(sizeof(double) * n3 * n3);
    ppo_xoshiro_normals(seed, G, n3 * n3); /* column-major fill (transforms.cpp:64-66) */
    rc = ppo_orthonormalize(G, n3, n3, F);
    if (!rc) memcpy(Q, F, sizeof(double) * n3 * p);
    free(G); free(F);
    return rc;
}

/* matrix_kernels.cpp:80-91 */
static void orthonormal_complement(const double* Q, int64_t n, int64_t p, double* C) {
    double* P = (double*)malloc(sizeof(double) * n * n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) P[i + j * n] = (i == j) ? 1.0 : 0.0;
    gemm('N', 'T', n, n, p, -1.0, Q, n, Q, n, 1.0, P, n);
    double* U = (double*)malloc(sizeof(double) * n * n);
    double* s = (double*)malloc(sizeof(double) * n);
    double* V = (double*)malloc(sizeof(double) * n * n);
    ppo_svd(P, n, n, U, s, V);
    memcpy(C, U, sizeof(double) * n * (n - p));
    free(P); free(U); free(s); free(V);
}

int ppo_data_dependent_q(const double* A, int64_t n1, int64_t n2, int64_t n3,
                         int64_t p, double* Q, double* sigma, int* completed) {
    int rc = check_dims(n3, p);
    if (rc) return rc;
    if (n1 < 1 || n2 < 1) return fail(PPO_SHAPE, "tensor extents must be positive");
    if (!all_finite(A, n1 * n2 * n3)) return fail(PPO_NUMERIC, "svd: input has non-finite entries");
    const int64_t N = n1 * n2;
    const int64_t avail = n3 < N ? n3 : N;
    double* U3 = (double*)malloc(sizeof(double) * n3 * avail);
    double* s = (double*)malloc(sizeof(double) * avail);
    if (N >= n3 && (double)N * n3 * n3 > 2e8) {
        /* unfolding (n3 x N) = tubes^T; tubes = Qt R  =>  U3 = right singular
         * vectors of R (n3 x n3). Same SVD as transforms.cpp:99, computed
         * through a QR preconditioner (as JacobiSVD itself does for
         * rectangular inputs). */
        double* T = (double*)malloc(sizeof(double) * N * n3);
        double* tau = (double*)malloc(sizeof(double) * n3);
        memcpy(T, A, sizeof(double) * N * n3);
        householder_qr(T, N, n3, tau);
        double* R = (double*)calloc((size_t)(n3 * n3), sizeof(double));
        for (int64_t j = 0; j < n3; ++j)
            for (int64_t i = 0; i <= j; ++i) R[i + j * n3] = T[i + j * N];
        free(T); free(tau);
        /* R = Ur S Vr^T ; unfolding = Vr S (Qt Ur)^T, so U3 = Vr */
        double* Ur = (double*)malloc(sizeof(double) * n3 * n3);
        double* Vr = (double*)malloc(sizeof(double) * n3 * n3);
        ppo_svd(R, n3, n3, Ur, s, Vr);
        memcpy(U3, Vr, sizeof(double) * n3 * n3);
        /* the sign rule belongs to the unfolding's U (matrix_kernels.cpp:35) */
        for (int64_t j = 0; j < n3; ++j) {
            int64_t imax = 0; double best = -1;
            for (int64_t i = 0; i < n3; ++i) { double a = fabs(U3[i + j * n3]); if (a > best) { best = a; imax = i; } }
            if (U3[imax + j * n3] < 0) for (int64_t i = 0; i < n3; ++i) U3[i + j * n3] = -U3[i + j * n3];
        }
        free(R); free(Ur); free(Vr);
    } else if (N >= n3) {
        /* Small case: one-sided Jacobi directly on the tube matrix T (N x n3);
         * its accumulated rotations are the unfolding's left singular vectors.
         * Like JacobiSVD, an already-orthogonal input is left unrotated, which
         * the degenerate 2x2x2 fixture pins (tests/test_decompositions.cpp:61-70). */
        double* W = (double*)malloc(sizeof(double) * N * n3);
        double* Vt = (double*)malloc(sizeof(double) * n3 * n3);
        memcpy(W, A, sizeof(double) * N * n3);
        hestenes(W, N, n3, Vt);
        double* sg = (double*)malloc(sizeof(double) * n3);
        int64_t* ord = (int64_t*)malloc(sizeof(int64_t) * n3);
        for (int64_t j = 0; j < n3; ++j) {
            double acc = 0;
            for (int64_t i = 0; i < N; ++i) acc += W[i + j * N] * W[i + j * N];
            sg[j] = sqrt(acc);
            ord[j] = j;
        }
        for (int64_t a = 1; a < n3; ++a) {
            int64_t x = ord[a], b = a - 1;
            while (b >= 0 && sg[ord[b]] < sg[x]) { ord[b + 1] = ord[b]; --b; }
            ord[b + 1] = x;
        }
        for (int64_t c = 0; c < n3; ++c) {
            s[c] = sg[ord[c]];
            memcpy(U3 + c * n3, Vt + ord[c] * n3, sizeof(double) * n3);
            int64_t imax = 0; double best = -1;
            for (int64_t i = 0; i < n3; ++i) { double a = fabs(U3[i + c * n3]); if (a > best) { best = a; imax = i; } }
            if (U3[imax + c * n3] < 0) for (int64_t i = 0; i < n3; ++i) U3[i + c * n3] = -U3[i + c * n3];
        }
        free(W); free(Vt); free(sg); free(ord);
    } else {
        double* unf = (double*)malloc(sizeof(double) * n3 * N);
        for (int64_t c = 0; c < N; ++c)
            for (int64_t k = 0; k < n3; ++k) unf[k + c * n3] = A[c + k * N];
        double* V = (double*)malloc(sizeof(double) * N * N);
        ppo_svd(unf, n3, N, U3, s, V);
        free(unf); free(V);
    }
    if (sigma) memcpy(sigma, s, sizeof(double) * (p < avail ? p : avail));
    if (p <= avail) {
        memcpy(Q, U3, sizeof(double) * n3 * p);
        if (completed) *completed = 0;
    } else {
        double* comp = (double*)malloc(sizeof(double) * n3 * (n3 - avail));
        orthonormal_complement(U3, n3, avail, comp);
        memcpy(Q, U3, sizeof(double) * n3 * avail);
        memcpy(Q + n3 * avail, comp, sizeof(double) * n3 * (p - avail));
        free(comp);
        if (completed) *completed = 1;
    }
    free(U3); free(s);
    return 0;
}

/* transforms.cpp:164-174: ||T - (T Q) Q^T||_F, computed directly. */
int ppo_projection_error(const double* A, int64_t n1, int64_t n2, int64_t n3,
                         const double* Q, int64_t p, double* err) {
    const int64_t N = n1 * n2;
    double* coeff = (double*)malloc(sizeof(double) * N * p);
    double* R = (double*)malloc(sizeof(double) * N * n3);
    gemm('N', 'N', N, p, n3, 1.0, A, N, Q, n3, 0.0, coeff, N);
    memcpy(R, A, sizeof(double) * N * n3);
    gemm('N', 'T', N, n3, p, -1.0, coeff, N, Q, n3, 1.0, R, N);
    *err = ppo_frobenius_norm(R, N * n3);
    free(coeff); free(R);
    return 0;
}

/* ---------------------------------------------------------- star products */
int ppo_star_q_product(const double* A, int64_t n1, int64_t m, int64_t n3,
                       const double* B, int64_t n2, const double* Q, int64_t p,
                       double scale, double* C) {
    if (n1 < 1 || m < 1 || n2 < 1 || n3 < 1 || p < 1)
        return fail(PPO_SHAPE, "star product: extents must be positive");
    /* star_products.cpp:51-59 */
    double* Ah = (double*)malloc(sizeof(double) * n1 * m * p);
    double* Bh = (double*)malloc(sizeof(double) * m * n2 * p);
    double* Ch = (double*)malloc(sizeof(double) * n1 * n2 * p);
    gemm('N', 'N', n1 * m, p, n3, 1.0, A, n1 * m, Q, n3, 0.0, Ah, n1 * m);
    gemm('N', 'N', m * n2, p, n3, 1.0, B, m * n2, Q, n3, 0.0, Bh, m * n2);
    ppo_facewise_product(Ah, n1, m, p, Bh, n2, Ch);
    gemm('N', 'T', n1 * n2, n3, p, 1.0, Ch, n1 * n2, Q, n3, 0.0, C, n1 * n2);
    if (scale != 1.0)
        for (int64_t i = 0; i < n1 * n2 * n3; ++i) C[i] *= scale;
    free(Ah); free(Bh); free(Ch);
    return 0;
}

/* ---------------------------------------------------------- decompositions */
typedef struct {
    const double* Ah;
    int64_t n1, n2, k, r;
    double *U, *S, *V;     /* truncated outputs (may be NULL) */
    double* s_all;         /* full spectra (r x p) (may be NULL) */
    int err;
} svd_ctx;
static void slice_svd_body(int64_t i, void* vctx) {
    svd_ctx* c = (svd_ctx*)vctx;
    const int64_t n1 = c->n1, n2 = c->n2, r = c->r, k = c->k;
    double* U = (double*)malloc(sizeof(double) * n1 * r);
    double* s = (double*)malloc(sizeof(double) * r);
    double* V = (double*)malloc(sizeof(double) * n2 * r);
    int rc = ppo_svd(c->Ah + i * n1 * n2, n1, n2, U, s, V);
    if (rc) c->err = rc;
    if (c->U) memcpy(c->U + i * n1 * k, U, sizeof(double) * n1 * k);
    if (c->V) memcpy(c->V + i * n2 * k, V, sizeof(double) * n2 * k);
    if (c->S) memcpy(c->S + i * k, s, sizeof(double) * k);
    if (c->s_all) memcpy(c->s_all + i * r, s, sizeof(double) * r);
    free(U); free(s); free(V);
}

int ppo_tsvdq(const double* A, int64_t n1, int64_t n2, int64_t n3,
              const double* Q, int64_t p, int64_t k, double* U, double* S, double* V) {
    /* decompositions.cpp:16-28 */
    const int64_t cap = n1 < n2 ? n1 : n2;
    if (k < 1 || k > cap) return fail(PPO_ARGUMENT, "tsvdq: k=%ld outside [1,%ld]", (long)k, (long)cap);
    const int64_t N = n1 * n2;
    double* Ah = (double*)malloc(sizeof(double) * N * p);
    gemm('N', 'N', N, p, n3, 1.0, A, N, Q, n3, 0.0, Ah, N); /* :65 A x3 Q^T */
    svd_ctx c = {Ah, n1, n2, k, cap, U, S, V, NULL, 0};
    parallel_for(p, slice_svd_body, &c);                      /* :75-81 */
    free(Ah);
    return c.err ? fail(c.err, "tsvdq: slice svd failed") : 0;
}

int ppo_slice_spectra(const double* A, int64_t n1, int64_t n2, int64_t n3,
                      const double* Q, int64_t p, double* s_all) {
    const int64_t N = n1 * n2, r = n1 < n2 ? n1 : n2;
    double* Ah = (double*)malloc(sizeof(double) * N * p);
    gemm('N', 'N', N, p, n3, 1.0, A, N, Q, n3, 0.0, Ah, N);
    svd_ctx c = {Ah, n1, n2, 1, r, NULL, NULL, NULL, s_all, 0};
    parallel_for(p, slice_svd_body, &c);
    free(Ah);
    return c.err;
}

typedef struct {
    const double *U, *S, *V;
    double* Ch;
    int64_t n1, n2, k;
} recon_ctx;
static void recon_body(int64_t i, void* vctx) {
    recon_ctx* c = (recon_ctx*)vctx;
    const int64_t n1 = c->n1, n2 = c->n2, k = c->k;
    double* US = (double*)malloc(sizeof(double) * n1 * k);
    for (int64_t j = 0; j < k; ++j)
        for (int64_t r = 0; r < n1; ++r) US[r + j * n1] = c->U[i * n1 * k + r + j * n1] * c->S[i * k + j];
    gemm('N', 'T', n1, n2, k, 1.0, US, n1, c->V + i * n2 * k, n2, 0.0, c->Ch + i * n1 * n2, n1);
    free(US);
}
int ppo_tsvdq_reconstruct(const double* U, const double* S, const double* V,
                          const double* Q, int64_t n1, int64_t n2, int64_t n3,
                          int64_t p, int64_t k, double* out) {
    const int64_t N = n1 * n2;
    double* Ch = (double*)malloc(sizeof(double) * N * p);
    recon_ctx c = {U, S, V, Ch, n1, n2, k};
    parallel_for(p, recon_body, &c);                                   /* :88-92 */
    gemm('N', 'T', N, n3, p, 1.0, Ch, N, Q, n3, 0.0, out, N);          /* :93 */
    free(Ch);
    return 0;
}

int ppo_tsvdq_error(const double* A, int64_t n1, int64_t n2, int64_t n3,
                    const double* U, const double* S, const double* V,
                    const double* Q, int64_t p, int64_t k,
                    double* total, double* eckart_young, double* projection) {
    const int64_t N = n1 * n2, r = n1 < n2 ? n1 : n2;
    /* :97-100 recompute all slice SVDs for the tail energies */
    double* s_all = (double*)malloc(sizeof(double) * r * p);
    int rc = ppo_slice_spectra(A, n1, n2, n3, Q, p, s_all);
    if (rc) { free(s_all); return rc; }
    double tail = 0.0;                                     /* :41-49 */
    for (int64_t i = 0; i < p; ++i)
        for (int64_t j = k; j < r; ++j) tail += s_all[j + i * r] * s_all[j + i * r];
    free(s_all);
    double* rec = (double*)malloc(sizeof(double) * N * n3);
    ppo_tsvdq_reconstruct(U, S, V, Q, n1, n2, n3, p, k, rec);
    double acc = 0.0;                                      /* :51-58 */
    for (int64_t i = 0; i < N * n3; ++i) { double d = A[i] - rec[i]; acc += d * d; }
    free(rec);
    *total = sqrt(acc);
    *eckart_young = sqrt(tail);
    return ppo_projection_error(A, n1, n2, n3, Q, p, projection);
}

int ppo_relative_error(const double* A, const double* Ahat, int64_t count, double* re) {
    const double ref = ppo_frobenius_norm(A, count);
    if (ref == 0.0) return fail(PPO_DEGENERATE, "relative_error: reference tensor is zero");
    double acc = 0.0;
    for (int64_t i = 0; i < count; ++i) { double d = A[i] - Ahat[i]; acc += d * d; }
    *re = sqrt(acc) / ref;
    return 0;
}

/* ------------------------------------------------------------- tsvdq2 */
typedef struct { double value; int64_t slice, pos; } pool_entry;
/* descending by value; ties by slice, then position (decompositions.cpp:148-150) */
static int pool_cmp(const void* x, const void* y) {
    const pool_entry* a = (const pool_entry*)x;
    const pool_entry* b = (const pool_entry*)y;
    if (a->value != b->value) return a->value > b->value ? -1 : 1;
    if (a->slice != b->slice) return a->slice < b->slice ? -1 : 1;
    if (a->pos != b->pos) return a->pos < b->pos ? -1 : 1;
    return 0;
}

int ppo_tsvdq2(const double* A, int64_t n1, int64_t n2, int64_t n3,
               const double* Q, int64_t p, double gamma,
               double* U, double* S, double* V, int64_t* multirank) {
    if (!(gamma > 0.0 && gamma <= 1.0))
        return fail(PPO_ARGUMENT, "tsvdq2: gamma must lie in (0,1], got %g", gamma);
    const int64_t N = n1 * n2, r = n1 < n2 ? n1 : n2;
    double* Ah = (double*)malloc(sizeof(double) * N * p);
    gemm('N', 'N', N, p, n3, 1.0, A, N, Q, n3, 0.0, Ah, N);
    /* full SVDs of every slice (decompositions.cpp:126) */
    svd_ctx c = {Ah, n1, n2, r, r, U, S, V, NULL, 0};
    parallel_for(p, slice_svd_body, &c);
    free(Ah);
    if (c.err) return fail(c.err, "tsvdq2: slice svd failed");
    /* pool of values above 1e-12 * global max (:137-145) */
    double gmax = 0.0;
    for (int64_t i = 0; i < p; ++i) if (S[i * r] > gmax) gmax = S[i * r];
    const double cutoff = 1e-12 * gmax;
    pool_entry* pool = (pool_entry*)malloc(sizeof(pool_entry) * (size_t)(p * r + 1));
    int64_t np = 0;
    for (int64_t i = 0; i < p; ++i)
        for (int64_t j = 0; j < r; ++j)
            if (S[j + i * r] > cutoff) pool[np++] = (pool_entry){S[j + i * r], i, j};
    qsort(pool, (size_t)np, sizeof(pool_entry), pool_cmp);
    /* prefix energy K (:154-167) */
    double total = 0.0;
    double* cum = (double*)malloc(sizeof(double) * (size_t)(np + 1));
    for (int64_t i = 0; i < np; ++i) { total += pool[i].value * pool[i].value; cum[i] = total; }
    int64_t K = 0;
    if (total > 0.0) {
        const double want = gamma * total;
        while (K < np && cum[K] < want) ++K;
        ++K;
        if (K > np) K = np;
    }
    for (int64_t i = 0; i < p; ++i) multirank[i] = 0;
    for (int64_t i = 0; i < K; ++i) multirank[pool[i].slice] += 1;
    /* keep the leading multirank[i] triplets, zero the rest */
    for (int64_t i = 0; i < p; ++i)
        for (int64_t j = multirank[i]; j < r; ++j) {
            S[j + i * r] = 0.0;
            for (int64_t q = 0; q < n1; ++q) U[q + (j + i * r) * n1] = 0.0;
            for (int64_t q = 0; q < n2; ++q) V[q + (j + i * r) * n2] = 0.0;
        }
    free(pool); free(cum);
    return 0;
}

int ppo_tsvdq2_error(const double* A, int64_t n1, int64_t n2, int64_t n3,
                     const double* U, const double* S, const double* V,
                     const double* Q, int64_t p, const int64_t* multirank,
                     double* total, double* eckart_young, double* projection) {
    const int64_t N = n1 * n2, r = n1 < n2 ? n1 : n2;
    double* s_all = (double*)malloc(sizeof(double) * r * p);
    int rc = ppo_slice_spectra(A, n1, n2, n3, Q, p, s_all);
    if (rc) { free(s_all); return rc; }
    double tail = 0.0;
    for (int64_t i = 0; i < p; ++i)
        for (int64_t j = multirank[i]; j < r; ++j) tail += s_all[j + i * r] * s_all[j + i * r];
    free(s_all);
    double* rec = (double*)malloc(sizeof(double) * N * n3);
    ppo_tsvdq_reconstruct(U, S, V, Q, n1, n2, n3, p, r, rec);
    double acc = 0.0;
    for (int64_t i = 0; i < N * n3; ++i) { double d = A[i] - rec[i]; acc += d * d; }
    free(rec);
    *total = sqrt(acc);
    *eckart_young = sqrt(tail);
    return ppo_projection_error(A, n1, n2, n3, Q, p, projection);
}
