/*
 * ppc.h — C-ABI of the B200-native projected star-Q / tSVDQ engine.
 *
 * Plain pointers and sizes, no torch or C++ types. Every entry point replaces
 * one function of the reference C++ API (/root/reference/proj/include/
 * projprod/ *.hpp); the citation is next to each declaration. The C++ API
 * mirror (include/projprod/ *.hpp, libprojprod.so) and the Python package
 * (paper_2409_19402_b200) are thin callers of these symbols.
 *
 * Conventions
 *   - FP64 everywhere; tensors are column-major, mode-1 fastest: entry
 *     (i,j,k) of an n1 x n2 x n3 tensor lives at i + j*n1 + k*n1*n2
 *     (tensor.hpp:13-19). The buffer is also the (n1*n2) x n3 tube matrix.
 *   - Matrices are column-major. A transform basis Q is n3 x p.
 *   - tSVDQ factor stacks are p contiguous column-major blocks: U (n1,k,p),
 *     V (n2,k,p), S (k,p) — the exported layout of tools/main.cpp:212-217
 *     and python/bindings.cpp:117-127.
 *   - `loc` says where ALL array pointers of one call live: PPC_HOST (the
 *     library copies in/out through the current stream) or PPC_DEVICE
 *     (pointers are device memory of the current device; results are
 *     stream-ordered and the call does not synchronize unless it returns a
 *     host scalar). Scalar outputs (double*) are always host pointers.
 *   - Caller-allocated outputs. Inputs are never modified.
 *   - Return codes map onto the reference's exception taxonomy
 *     (errors.hpp:9-37); ppc_last_error() holds the message (thread-local).
 *   - Calls are reentrant across host threads; each thread has its own
 *     current device and stream (ppc_set_device / ppc_set_stream).
 */
#ifndef PPC_H
#define PPC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPC_VERSION 1

typedef enum {
    PPC_OK = 0,
    PPC_SHAPE = 1,       /* shape_error            (errors.hpp:10-12) */
    PPC_BOUNDS = 2,      /* bounds_error           (errors.hpp:15-17) */
    PPC_ARGUMENT = 3,    /* argument_error         (errors.hpp:20-22) */
    PPC_DEGENERATE = 4,  /* degenerate_input_error (errors.hpp:26-28) */
    PPC_NUMERIC = 5,     /* numeric_error          (errors.hpp:31-33) */
    PPC_FORMAT = 6,      /* format_error           (errors.hpp:36-38) */
    PPC_CUDA = 7,        /* CUDA / NCCL runtime failure (no reference analogue) */
    PPC_NO_DEVICE = 8    /* no usable sm_100 device: the engine has no CPU path */
} ppc_status;

enum { PPC_HOST = 0, PPC_DEVICE = 1 };

const char* ppc_last_error(void);
int ppc_version(void);

/* ---- runtime ----------------------------------------------------------- */
/* Number of visible CUDA devices (0 when none). PROJPROD_DEVICES caps it,
 * mirroring PROJPROD_THREADS (parallel.cpp:13-27). */
int ppc_device_count(void);
int ppc_set_device(int device);
/* Stream (cudaStream_t) used by this thread's subsequent calls. NULL selects
 * the legacy default stream (what torch reports as stream 0). Until the first
 * call the library uses its own non-blocking stream. */
int ppc_set_stream(void* stream);
void* ppc_get_stream(void);
int ppc_synchronize(void);
/* Release this thread's cached large device workspaces (blocks >= 256 MB that
 * the library keeps between calls of the same shapes) on the current device.
 * Engine extension: the CPU reference has no device memory to trim. */
int ppc_trim_workspace(void);
/* Kernel launches issued by the library on this thread since the last reset
 * (for the bench's gpu_launches count). */
int64_t ppc_launch_count(int reset);
/* Per-stage device timing with CUDA events recorded on the launching stream
 * (off by default). ppc_timing_report writes a JSON object
 * {"stage": {"ms", "n", "flops", "bytes"}} (algorithmic flops/bytes). */
int ppc_timing_enable(int on);
/* GEMM kernel selection: 0 = automatic (warp-specialized TMA kernel where
 * eligible), 1 = always the cp.async kernel. Both accumulate every output in
 * the same order, so results are bitwise identical (used by the tests). */
int ppc_set_gemm_path(int mode);
/* Arithmetic of the large products: 1 = automatic (default): the FP64 Gram
 * SYRKs, the compress chain's forward transform, the slice-SVD filter /
 * Rayleigh-Ritz products, the reconstruction residual and the star-Q facewise
 * product run on the INT8 tensor cores as FP64 emulation (Ozaki digit
 * splitting, 6-7 digits, where eligible; the facewise product only for
 * operands that pass the dynamic-range gate), the rest on FP64 DMMA;
 * 0 = every product on FP64 DMMA (the FP64-only switch). PPC_OZAKI=0 in the
 * environment sets 0. Results agree to ~1e-14 relative (not bitwise).
 * ppc_get_ozaki returns the current mode. */
int ppc_set_ozaki(int mode);
int ppc_get_ozaki(void);
/* The batched Ozaki SYRK on DEVICE memory (test hook for the INT8 path):
 * G_b = A_b^T A_b (n x n) for A_b = A + b*strideA (rows x n, lda),
 * 1024 <= rows <= 4096, n >= 128. PPC_ARGUMENT when not eligible. */
int ppc_ozaki_syrk_batched(const double* A, int64_t lda, int64_t strideA, int64_t rows, int64_t n, int64_t batch,
                           double* G);
int ppc_timing_report(char* buf, int64_t cap, int reset);

/* ---- L3 kernels (tensor.hpp, matrix_kernels.hpp) ------------------------ */
/* tensor.hpp:87 / tensor.cpp:139-147: out = A x3 op(M).
 * trans_m = 0: M is q x n3 (out tube matrix = T * M^T).
 * trans_m = 1: M is n3 x q (out = A x3 M^T = T * M), the forward transform
 * with Q passed directly (no Q^T copy, cf. decompositions.cpp:65). */
int ppc_mode3_product(const double* A, int64_t n1, int64_t n2, int64_t n3,
                      const double* M, int64_t q, int trans_m, double* out, int loc);

/* tensor.hpp:84 / tensor.cpp:109-137: out = A x_mode M, M is q x n_mode
 * (column-major); the mode's extent becomes q. mode 3 is ppc_mode3_product
 * with trans_m = 0; modes 1 and 2 serve the HOSVD baseline. */
int ppc_mode_product(const double* A, int64_t n1, int64_t n2, int64_t n3,
                     const double* M, int64_t q, int mode, double* out, int loc);

/* tensor.hpp:90 / tensor.cpp:149-156: C(:,:,k) = A(:,:,k) B(:,:,k);
 * A n1 x m x n3, B m x n2 x n3, C n1 x n2 x n3. */
int ppc_facewise_product(const double* A, int64_t n1, int64_t m, int64_t n3,
                         const double* B, int64_t n2, double* C, int loc);

/* tensor.hpp:92 / tensor.cpp:158 (deterministic fixed-order reduction). */
int ppc_frobenius_norm(const double* A, int64_t count, double* out, int loc);

/* matrix_kernels.hpp:19-22 / matrix_kernels.cpp:29-46: batched thin SVD,
 * keeping the leading k triplets (k = min(m,n) for svd(), 1 <= k for
 * truncated_svd()). A is `batch` contiguous m x n blocks; U (m,k,batch),
 * s (k,batch), V (n,k,batch). Sign rule of matrix_kernels.cpp:16-25. */
int ppc_svd_batched(const double* A, int64_t m, int64_t n, int64_t batch, int64_t k,
                    double* U, double* s, double* V, int loc);

/* ---- L4 transforms (transforms.hpp) ------------------------------------- */
/* transforms.hpp:49 / transforms.cpp:97-115: Q = U3(:,1:p) of the mode-3
 * unfolding (Gram SYRK + symmetric top-p eigensolve on the device, sign rule
 * on each column). sigma (nullable, host or device per loc) receives the p
 * leading singular values of the unfolding; *completed (host, nullable) is
 * set when p > min(n3, n1*n2) forced an orthonormal completion. */
int ppc_data_dependent_q(const double* A, int64_t n1, int64_t n2, int64_t n3,
                         int64_t p, double* Q, double* sigma, int* completed, int loc);

/* transforms.hpp:67 / transforms.cpp:164-174: ||A - A x3 QQ^T||_F. */
int ppc_projection_error(const double* A, int64_t n1, int64_t n2, int64_t n3,
                         const double* Q, int64_t p, double* err, int loc);

/* Host-side builders of the structured bases (tiny; transforms.cpp:33-95). */
int ppc_dct_q(int64_t n3, int64_t p, double* Q);                          /* host */
int ppc_haar_q(int64_t n3, int64_t p, double* Q);                         /* host */
int ppc_random_orthogonal_q(int64_t n3, int64_t p, uint64_t seed, double* Q); /* host */
int ppc_identity_q(int64_t n3, int64_t p, double* Q);                     /* host */
/* matrix_kernels.cpp:48-78 orthonormalize (rank gate, Householder QR, sign rule). */
int ppc_orthonormalize(const double* A, int64_t n, int64_t p, double* Q);    /* host */
/* transforms.cpp:20-27 + 100-109 of custom_transform: Stiefel check. */
int ppc_check_stiefel(const double* Q, int64_t n3, int64_t p);            /* host */

/* ---- L5 drivers (star_products.hpp, decompositions.hpp, metrics.hpp) ----- */
/* star_products.hpp:28 / star_products.cpp:51-59:
 * C = [(A x3 Q^T) facewise (B x3 Q^T)] x3 Q, times scale. */
int ppc_star_q_product(const double* A, int64_t n1, int64_t m, int64_t n3,
                       const double* B, int64_t n2, const double* Q, int64_t p,
                       double scale, double* C, int loc);

/* decompositions.hpp:90 / decompositions.cpp:62-83. */
int ppc_tsvdq(const double* A, int64_t n1, int64_t n2, int64_t n3,
              const double* Q, int64_t p, int64_t k,
              double* U, double* S, double* V, int loc);

/* decompositions.hpp:91 / decompositions.cpp:85-94. */
int ppc_tsvdq_reconstruct(const double* U, const double* S, const double* V,
                          const double* Q, int64_t n1, int64_t n2, int64_t n3,
                          int64_t p, int64_t k, double* out, int loc);

/* decompositions.hpp:92 / decompositions.cpp:96-103: (total, eckart_young,
 * projection). total is measured directly against the reconstruction (fused
 * on the device, never materialized); eckart_young comes from fresh slice
 * SVDs of A x3 Q^T as in the reference. */
int ppc_tsvdq_error(const double* A, int64_t n1, int64_t n2, int64_t n3,
                    const double* U, const double* S, const double* V,
                    const double* Q, int64_t p, int64_t k,
                    double* total, double* eckart_young, double* projection, int loc);

/* metrics.hpp:21 / metrics.cpp:21-28: ||A - Ahat|| / ||A||. */
int ppc_relative_error(const double* A, const double* Ahat, int64_t count,
                       double* re, int loc);

/* Fused relative_error(A, tsvdq_reconstruct(F)) without materializing the
 * reconstruction (tools/main.cpp:276-283 call chain). */
int ppc_tsvdq_relative_error(const double* A, int64_t n1, int64_t n2, int64_t n3,
                             const double* U, const double* S, const double* V,
                             const double* Q, int64_t p, int64_t k,
                             double* re, int loc);

/* ---- tsvdq2: energy-truncated multirank ------------------ */
/* decompositions.cpp:120-190 tsvdq2(A, T, gamma), gamma in (0,1]. Full
 * transform-domain spectra on the device; the global descending sort (ties
 * by slice, then position) and the prefix-energy cut over the p*r values on
 * the host. The ragged per-slice factors of TsvdqIIFactors
 * (decompositions.hpp:45-56) are returned padded to r = min(n1,n2) columns:
 * U (n1,r,p), S (r,p), V (n2,r,p), zero beyond multirank[i]. multirank is a
 * HOST array of p entries in every mode (it is bookkeeping, not data). */
int ppc_tsvdq2(const double* A, int64_t n1, int64_t n2, int64_t n3,
               const double* Q, int64_t p, double gamma,
               double* U, double* S, double* V, int64_t* multirank, int loc);
/* decompositions.cpp:192-201 on the padded factors above. */
int ppc_tsvdq2_reconstruct(const double* U, const double* S, const double* V,
                           const double* Q, int64_t n1, int64_t n2, int64_t n3,
                           int64_t p, const int64_t* multirank, double* out, int loc);
/* decompositions.cpp:203-209: eckart_young from fresh full spectra with the
 * per-slice multirank; total fused as in ppc_tsvdq_error. */
int ppc_tsvdq2_error(const double* A, int64_t n1, int64_t n2, int64_t n3,
                     const double* U, const double* S, const double* V,
                     const double* Q, int64_t p, const int64_t* multirank,
                     double* total, double* eckart_young, double* projection, int loc);

/* ---- star-M product and the Tucker / flattened baselines -- */
/* star_products.cpp:38-49: C = [(A x3 M) facewise (B x3 M)] x3 M^{-1} for an
 * invertible n3 x n3 M (PPC_DEGENERATE when numerically singular:
 * numerical rank at 1e-12 below n3). A n1 x m x n3, B m x n2 x n3. */
int ppc_star_m_product(const double* A, int64_t n1, int64_t m, int64_t n3,
                       const double* B, int64_t n2, const double* M, double* C, int loc);
/* decompositions.cpp:211-236 hosvd(A, k1, k2, k3): mode factors from the
 * unfolding Grams (top eigenvectors, sign rule), core = A x1 U1^T x2 U2^T
 * x3 U3^T. 1 <= ki <= ni (PPC_ARGUMENT otherwise). */
int ppc_hosvd(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t k1, int64_t k2,
              int64_t k3, double* core, double* U1, double* U2, double* U3, int loc);
/* decompositions.cpp:238-242 */
int ppc_hosvd_reconstruct(const double* core, int64_t k1, int64_t k2, int64_t k3,
                          const double* U1, int64_t n1, const double* U2, int64_t n2,
                          const double* U3, int64_t n3, double* out, int loc);
/* decompositions.cpp:244-255 matrix_svd_baseline(A, k): rank-k SVD of the
 * (n1 n3) x n2 stack of frontal slices; U ((n1 n3) x k), s (k), V (n2 x k),
 * *error = ||B - U diag(s) V^T||_F measured directly. */
int ppc_matrix_svd_baseline(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t k,
                            double* U, double* s, double* V, double* error, int loc);

/* ---- PT3 container I/O (io.hpp:11-30, io.cpp:52-112) ------ */
/* Header: "PT3\0", u32 version 1, u8 dtype 1 (float64), u8 flags 0, 2 pad,
 * u64 n1, n2, n3 (little endian), then the mode-1-fastest payload, which is
 * the engine's tensor layout. Malformed files (magic, version, dtype, flags,
 * zero extent, overflowing extents, truncated or trailing bytes) fail with
 * PPC_FORMAT, as read_pt3 throws format_error. Device reads and writes stream
 * through two pinned staging buffers on the copy stream, overlapping disk and
 * PCIe; host calls are plain file I/O and need no GPU. */
int ppc_pt3_info(const char* path, int64_t* n1, int64_t* n2, int64_t* n3);
/* count must equal n1*n2*n3 of the file (PPC_SHAPE otherwise). */
int ppc_pt3_read(const char* path, double* dst, int64_t count, int loc);
int ppc_pt3_write(const char* path, const double* src, int64_t n1, int64_t n2, int64_t n3, int loc);

/* ---- shard-level building blocks (multi-GPU driver, dist.py) ------------ */
/* Deterministic Gram plan for a tube matrix of N rows and n3 columns: the
 * number of row chunks (a power of two) and the chunk length. Depends on
 * (N, n3) only, so a pixel-sharded run reproduces the 1-GPU sums bitwise. */
int ppc_gram_plan(int64_t N, int64_t n3, int64_t* chunks, int64_t* chunk);
/* Strided batched FP64 GEMM on DEVICE memory, the sharded star-Q driver's
 * building block (facewise GEMM into a lateral block of the output slices;
 * inverse transform with the scale folded into the epilogue, as
 * star_products.cpp:56-58 applies it):
 *   C_b = alpha * op(A_b) * op(B_b),  b < batch,
 * op(A) = A (M x K, lda) or, trans_a, A^T with A stored K x M (lda);
 * op(B) = B (K x N, ldb) or, trans_b, B^T with B stored N x K (ldb);
 * X_b = X + b * strideX. Same DMMA kernels and accumulation order as the
 * engine's own mode-3 / facewise stages. */
int ppc_gemm_strided(int64_t M, int64_t N, int64_t K, int64_t batch, double alpha,
                     const double* A, int64_t lda, int64_t strideA, int trans_a,
                     const double* B, int64_t ldb, int64_t strideB, int trans_b,
                     double* C, int64_t ldc, int64_t strideC);
/* ---- multi-GPU building blocks (paper_2409_19402_b200/dist.py) ----------- */
/* Facewise product of one slice group into a strided output, DEVICE memory,
 * stream-ordered: C(:,:,i) (at C + i*strideC, leading dimension ldc) =
 * A(:,:,i) B(:,:,i), A n1 x m x batch and B m x n2 x batch contiguous. Runs
 * on the INT8 tensor cores when star_q's facewise would (256 <= m <= 4096,
 * rows in whole 128-row blocks, operands passing the dynamic-range gate),
 * else on FP64 DMMA: the row-sharded star-Q's replacement of
 * tensor.cpp:149-156 for the rank's C rows. */
int ppc_facewise_strided(const double* A, int64_t n1, int64_t m, int64_t batch, const double* B, int64_t n2,
                         double* C, int64_t ldc, int64_t strideC);
/* The star product's inverse transform, DEVICE memory, stream-ordered:
 * C (N x n3, column-major) = scale Ch Q^T for Ch (N x p) and Q (n3 x p) --
 * what star_q runs for C^ x3 Q (star_products.cpp:56-58). On the INT8 tensor
 * cores with one scale per row of Ch (rows are independent: a row shard gives
 * the 1-GPU bits) when 32 <= p <= 64 and n3 <= 256 is a multiple of 32, else
 * FP64 DMMA. The row-sharded star-Q's inverse transform. */
int ppc_star_inverse(const double* Ch, int64_t N, int64_t p, const double* Q, int64_t n3, double scale, double* C);
/* The pixel -> slice reshard's unpack, DEVICE memory, stream-ordered:
 * recv holds G blocks [r][slice][j][i] (rank r's nj lateral columns of my ps
 * slices, as all_to_all_single delivers them); out receives the ps whole
 * n1 x (G nj) slices [slice][r nj + j][i] that the slice SVDs read. */
int ppc_reshard_slices(const double* recv, int64_t G, int64_t ps, int64_t nj, int64_t n1, double* out);
/* Partial Grams T_c^T T_c of `nchunks` consecutive chunks of `chunk` rows of
 * T (rows x n3, leading dimension ldT): parts is nchunks x n3 x n3. */
int ppc_gram_partials(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk,
                      int64_t nchunks, double* parts, int loc);
/* As ppc_gram_partials on device memory, and when the INT8 path splits T into
 * whole 4096-row blocks it keeps T's 7-digit split in the engine: *handle > 0
 * names it (0: nothing kept). ppc_mode3_forward_digits then forms T Q from the
 * kept digits on the INT8 tensor cores (the sharded forward transform), and
 * ppc_digits_release frees them. Handles belong to the calling thread.
 * *nonfinite (host) = 1 when T holds a NaN or Inf (the shard's half of
 * matrix_kernels.cpp:32; the multi-GPU driver combines it over the ranks and
 * raises PPC_NUMERIC on every one of them), else 0. */
int ppc_gram_partials_keep(const double* T, int64_t ldT, int64_t rows, int64_t n3, int64_t chunk,
                           int64_t nchunks, double* parts, int64_t* handle, int* nonfinite);
/* out (rows x p, leading dimension rows, device) = T Q (Q: n3 x p, device) from
 * the digits kept under handle; PPC_ARGUMENT when the handle is unknown or the
 * shape does not qualify (the caller then uses ppc_mode3_product). */
int ppc_mode3_forward_digits(int64_t handle, const double* Q, int64_t p, double* out);
int ppc_digits_release(int64_t handle);
/* parts[0] = fixed pairwise tree sum of nparts arrays of `elems` doubles. */
int ppc_tree_reduce(double* parts, int64_t nparts, int64_t elems, int loc);
/* The same eigensolve split across ranks, DEVICE memory, stream-ordered:
 * _begin tridiagonalizes G (n x n; replicated on every rank) and returns a
 * handle (0: the size takes another solver; use ppc_sym_eig_top);
 * _vectors writes the inverse-iteration vectors of eigenvalues j0..j1-1
 * (0 = largest) to Z (n x (j1-j0)); the caller gathers all p of them into
 * Zall (n x p); _finish orthonormalizes Zall (in place, replicated) and
 * writes columns j0..j1-1 of Q (sign rule applied) to Q (n x (j1-j0)).
 * Q is bitwise the ppc_sym_eig_top result for any split. Handles belong to
 * the calling thread; _release frees one. */
int ppc_sym_eig_split_begin(const double* G, int64_t n, int64_t p, int64_t* handle);
int ppc_sym_eig_split_vectors(int64_t handle, int64_t j0, int64_t j1, double* Z);
int ppc_sym_eig_split_finish(int64_t handle, double* Zall, int64_t j0, int64_t j1, double* Q);
int ppc_sym_eig_split_release(int64_t handle);
/* Top-p eigenvectors Q (n x p, sign rule) and sigma = sqrt(lambda) (nullable)
 * of the symmetric PSD Gram G (n x n): the tail of data_dependent_transform. */
int ppc_sym_eig_top(const double* G, int64_t n, int64_t p, double* Q, double* sigma, int loc);
/* sums[0..1] (host) = {sum_i ||A_i - U_i diag(S_i) V_i^T||^2, sum_i ||A_i||^2} over
 * `batch` transform-domain slices A_i (n1 x n2, stride n1*n2) and their rank-k
 * factors U (n1,k,batch), S (k,batch), V (n2,k,batch): the slice-space half of
 * the orthogonal split of ||A - A_k||^2 (relative_error of the compress chain,
 * metrics.cpp:21-28; the sharded driver sums it over the slice shards). */
int ppc_slice_residual_sums(const double* A, int64_t n1, int64_t n2, int64_t batch, int64_t k,
                            const double* U, const double* S, const double* V, double* sums, int loc);
/* *trace (host) = trace of the n x n matrix G (fixed summation order): ||T||_F^2
 * from the data-driven Q's Gram G = T^T T. */
int ppc_gram_trace(const double* G, int64_t n, double* trace, int loc);
/* {sum (A - recon)^2, sum A^2} over a lateral block of pixels: A_blk is the
 * n1 x nj x n3 block of columns [j0, j0+nj) (leading dims n1 and ldA = n1*n2
 * between frontal slices), U (n1,k,p), S (k,p), V (n2,k,p) full factors. */
int ppc_recon_residual_block(const double* A_blk, int64_t n1, int64_t nj, int64_t n3,
                             int64_t ldA, const double* U, const double* S, const double* V,
                             int64_t n2, int64_t j0, const double* Q, int64_t p, int64_t k,
                             double* sums, int loc);

/* The `projprod sweep` loop (tools/main.cpp:299-341: relative error of the
 * rank-k tSVDQ over a grid of (p, k)), amortized: one basis at
 * max p (data-dependent bases of smaller p are its leading columns, exactly
 * as data_dependent_transform(A, p) = U3(:,1:p); cf. verify.cpp:1149-1158),
 * one slice SVD per transform-domain slice at max k (slice i does not depend
 * on p), then one fused residual pass per (p, k). Q (n3 x max p) is used
 * when non-null, else the data-driven basis is built. re (nk x np,
 * column-major): re[ik + ip*nk]. Extents in ps / ks are host arrays. */
int ppc_tsvdq_sweep(const double* A, int64_t n1, int64_t n2, int64_t n3, const int64_t* ps,
                    int64_t np, const int64_t* ks, int64_t nk, const double* Q, double* re, int loc);

/* The `projprod compress --method tsvdq --transform data` pipeline
 * (tools/main.cpp:186-283: data_dependent_transform -> tsvdq ->
 * tsvdq_reconstruct -> relative_error) as one call: A is staged once, the
 * reconstruction is never materialized. Q (n3,p), sigma (p, nullable),
 * U (n1,k,p), S (k,p), V (n2,k,p); *re = ||A - recon|| / ||A||. */
int ppc_tsvdq_compress(const double* A, int64_t n1, int64_t n2, int64_t n3, int64_t p,
                       int64_t k, double* Q, double* sigma, double* U, double* S, double* V,
                       double* re, int loc);

#ifdef __cplusplus
}
#endif
#endif /* PPC_H */
