/*
 * ppo — CPU oracle for the projected star-Q product and truncated tSVDQ.
 *
 * TEST INFRASTRUCTURE ONLY. This is a plain-C restatement of the reference
 * C++/Eigen implementation (/root/reference/proj) used as the parity checker
 * by tests/, by __graft_entry__.smoke() and as the CPU baseline leg of
 * bench.py. The product path (paper_2409_19402_b200/, include/ppc.h) never
 * links or calls it.
 *
 * Conventions (mirroring proj/include/projprod/tensor.hpp:13-19):
 *   - all doubles, column-major, mode-1 fastest: entry (i,j,k) of an
 *     n1 x n2 x n3 tensor lives at i + j*n1 + k*n1*n2;
 *   - a transform basis Q is n3 x p column-major;
 *   - tSVDQ factor stacks are p contiguous column-major blocks: U is
 *     (n1,k,p), V is (n2,k,p), S is (k,p) — the exported layout of
 *     proj/tools/main.cpp:212-217 and proj/python/bindings.cpp:117-127.
 *   - return codes mirror proj/include/projprod/errors.hpp:9-37:
 *     0 ok, 1 shape, 2 bounds, 3 argument, 4 degenerate, 5 numeric.
 */
#ifndef PPO_H
#define PPO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PPO_OK = 0, PPO_SHAPE = 1, PPO_BOUNDS = 2, PPO_ARGUMENT = 3,
       PPO_DEGENERATE = 4, PPO_NUMERIC = 5 };

const char* ppo_last_error(void);
void ppo_set_threads(int n);   /* 0 = PROJPROD_THREADS / hardware default */
int ppo_threads(void);
/* Optional: route GEMMs through an OpenBLAS dgemm (e.g. SciPy's bundled
 * libscipy_openblas) loaded with dlopen; symbol is the dgemm_ name in it.
 * Used only to make the CPU baseline's GEMM comparable to Eigen's. */
int ppo_use_blas(const char* lib_path, const char* dgemm_symbol,
                 const char* set_threads_symbol);
int ppo_set_blas_threads(int n);

/* tensor.cpp:139-147  out.tubes = A.tubes * M^T, M is q x n3. */
int ppo_mode3_product(const double* A, int64_t n1, int64_t n2, int64_t n3,
                      const double* M, int64_t q, double* out);
/* tensor.cpp:149-156  C(:,:,k) = A(:,:,k) * B(:,:,k), A n1 x m x n3, B m x n2 x n3. */
int ppo_facewise_product(const double* A, int64_t n1, int64_t m, int64_t n3,
                         const double* B, int64_t n2, double* C);
/* tensor.cpp:158 */
double ppo_frobenius_norm(const double* A, int64_t count);

/* matrix_kernels.cpp:15-37  thin SVD r=min(m,n), descending s, sign rule. */
int ppo_svd(const double* A, int64_t m, int64_t n, double* U, double* s, double* V);
/* matrix_kernels.cpp:48-78 */
int ppo_orthonormalize(const double* A, int64_t n, int64_t p, double* Q);

/* transforms.cpp:33-43,89-95 */
int ppo_dct_q(int64_t n3, int64_t p, double* Q);
/* transforms.cpp:62-68,80-87 */
int ppo_random_orthogonal_q(int64_t n3, int64_t p, uint64_t seed, double* Q);
/* transforms.cpp:97-115  Q = U3(:,1:p); *completed set when padded. */
int ppo_data_dependent_q(const double* A, int64_t n1, int64_t n2, int64_t n3,
                         int64_t p, double* Q, double* sigma, int* completed);
/* transforms.cpp:164-174 */
int ppo_projection_error(const double* A, int64_t n1, int64_t n2, int64_t n3,
                         const double* Q, int64_t p, double* err);

/* star_products.cpp:51-59 */
int ppo_star_q_product(const double* A, int64_t n1, int64_t m, int64_t n3,
                       const double* B, int64_t n2, const double* Q, int64_t p,
                       double scale, double* C);

/* decompositions.cpp:62-83 */
int ppo_tsvdq(const double* A, int64_t n1, int64_t n2, int64_t n3,
              const double* Q, int64_t p, int64_t k,
              double* U, double* S, double* V);
/* decompositions.cpp:85-94 */
int ppo_tsvdq_reconstruct(const double* U, const double* S, const double* V,
                          const double* Q, int64_t n1, int64_t n2, int64_t n3,
                          int64_t p, int64_t k, double* out);
/* decompositions.cpp:96-103 (+ helpers :30-58) */
int ppo_tsvdq_error(const double* A, int64_t n1, int64_t n2, int64_t n3,
                    const double* U, const double* S, const double* V,
                    const double* Q, int64_t p, int64_t k,
                    double* total, double* eckart_young, double* projection);
/* All transform-domain singular values (full spectra), r = min(n1,n2):
 * s_all is (r, p). Used by tests for tail energies and tsvdq2. */
int ppo_slice_spectra(const double* A, int64_t n1, int64_t n2, int64_t n3,
                      const double* Q, int64_t p, double* s_all);
/* decompositions.cpp:120-209 tsvdq2: energy-truncated multirank. Factor
 * stacks are padded to r = min(n1,n2) columns per slice (zero beyond
 * multirank[i]); multirank has p entries. */
int ppo_tsvdq2(const double* A, int64_t n1, int64_t n2, int64_t n3,
               const double* Q, int64_t p, double gamma,
               double* U, double* S, double* V, int64_t* multirank);
/* decompositions.cpp:344-350: tail energies with the per-slice multirank. */
int ppo_tsvdq2_error(const double* A, int64_t n1, int64_t n2, int64_t n3,
                     const double* U, const double* S, const double* V,
                     const double* Q, int64_t p, const int64_t* multirank,
                     double* total, double* eckart_young, double* projection);
/* metrics.cpp:21-28 */
int ppo_relative_error(const double* A, const double* Ahat, int64_t count,
                       double* re);

/* rng.hpp:30-80  xoshiro256++ Box-Muller normals in buffer order. */
void ppo_xoshiro_normals(uint64_t seed, double* out, int64_t count);
uint64_t ppo_derive_seed(uint64_t seed, uint64_t stream);

#ifdef __cplusplus
}
#endif
#endif
