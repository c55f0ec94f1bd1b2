"""CPU baseline of the compress chain at the full BASELINE config, on LAPACK.

TEST / BENCH INFRASTRUCTURE ONLY (like ppo.py): used by bench.py's
cpu_baseline and --impl reference legs, and pinned against the C oracle by
tests/test_oracle_kat.py. Never imported by the product package.

The reference chain (`compress --method tsvdq --transform data`,
tools/main.cpp:186-283) is restated step by step, with LAPACK/BLAS (numpy's
OpenBLAS, all host threads) for the dense kernels, because the C oracle's
one-sided Jacobi -- the faithful restatement of Eigen's JacobiSVD -- needs
~25 s for one 1024^2 matrix and ~200 s for one 2048^2 slice on one core,
which no bounded sample can hold:

  1. data_dependent_transform (transforms.cpp:97-115): the left singular
     vectors of the n3 x N unfolding = the right singular vectors of the
     N x n3 tube matrix T, via T = QR (dgeqrf) and the SVD of R (dgesdd);
  2. tsvdq (decompositions.cpp:62-83): Ahat = T Q (dgemm), then the
     rank-k truncation of every n1 x n2 frontal slice (dgesdd);
  3. tsvdq_reconstruct + relative_error (decompositions.cpp:85-94,
     metrics.cpp:21-28): C_i = U_i S_i V_i^T, A_k = C x3 Q, ||A - A_k|| / ||A||.

dgesdd is much faster than the reference's Jacobi SVD, so the baseline is
optimistic for the CPU (conservative for the GPU ratio).

Timing a full cfg5 step (2048 x 2048 x 1024, 32 GiB) is not bounded, so
`compress_timed` runs the same steps on a lateral pixel subsample for the
parts linear in N (QR, transforms, reconstruction, residual) and on `nslices`
whole n1 x n2 slices of the same distribution for the slice SVDs, and
extrapolates linearly in N and in p. The SVD of R
(n3 x n3) does not depend on N and is timed whole.
"""
from __future__ import annotations

import time

import numpy as np


def data_q(T: np.ndarray, p: int) -> np.ndarray:
    """Top-p left singular vectors of the unfolding (= right singular vectors
    of T), the reference's sign rule (matrix_kernels.cpp:16-25) applied."""
    R = np.linalg.qr(T, mode="r")
    _, _, vt = np.linalg.svd(R, full_matrices=False)
    q = vt[:p].T.copy()
    for j in range(p):
        i = int(np.argmax(np.abs(q[:, j])))
        if q[i, j] < 0:
            q[:, j] *= -1
    return np.asfortranarray(q)


def truncated(sl: np.ndarray, k: int):
    u, s, vt = np.linalg.svd(sl, full_matrices=False)
    return u[:, :k], s[:k], vt[:k].T


def compress(a: np.ndarray, p: int, k: int):
    """The whole chain on a host tensor (n1, n2, n3): (Q, U, S, V, RE)."""
    n1, n2, n3 = a.shape
    T = a.reshape(n1 * n2, n3, order="F")
    q = data_q(T, p)
    ah = T @ q
    U, S, V = np.zeros((n1, k, p)), np.zeros((k, p)), np.zeros((n2, k, p))
    ch = np.empty_like(ah)
    for i in range(p):
        u, s, v = truncated(ah[:, i].reshape(n1, n2, order="F"), k)
        U[:, :, i], S[:, i], V[:, :, i] = u, s, v
        ch[:, i] = ((u * s) @ v.T).reshape(-1, order="F")
    rec = ch @ q.T
    re = np.linalg.norm(T - rec) / np.linalg.norm(T)
    return q, U, S, V, re


def compress_timed(gen_block, n1: int, n2: int, n3: int, p: int, k: int, nj: int, gen_slice,
                   nslices: int = 1):
    """Extrapolated seconds of one full compress step.

    gen_block(nj) -> the lateral block A[:, :nj, :] (n1, nj, n3) of the
    workload's distribution (the N-linear sample: N_s = n1 nj pixels);
    gen_slice(i) -> one n1 x n2 transform-domain slice of the same kind.
    Returns (seconds, detail dict)."""
    blk = gen_block(nj)  # (callers may cache the sample: generation is not timed)
    Ns, N = n1 * nj, n1 * n2
    T = blk.reshape(Ns, n3, order="F")
    t0 = time.perf_counter()
    R = np.linalg.qr(T, mode="r")                    # transforms.cpp:99 (QR part)
    t_qr = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, _, vt = np.linalg.svd(R, full_matrices=False)  # SVD of R (N-independent)
    t_rsvd = time.perf_counter() - t0
    q = np.asfortranarray(vt[:p].T)
    t0 = time.perf_counter()
    ah = T @ q                                       # decompositions.cpp:65
    t_fwd = time.perf_counter() - t0
    sl = [gen_slice(i) for i in range(nslices)]  # not timed
    t0 = time.perf_counter()
    fac = [truncated(x, k) for x in sl]              # decompositions.cpp:75-81
    t_svd = (time.perf_counter() - t0) / nslices
    # reconstruction of the sample's pixels: C_i restricted to the block's
    # lateral columns (U_i S_i V_i[:nj]^T), A_k = C Q^T, and the residual
    u, s, v = fac[0]
    t0 = time.perf_counter()
    ch = np.empty((Ns, p))
    for i in range(p):
        ch[:, i] = ((u * s) @ v[:nj].T).reshape(-1, order="F")
    rec = ch @ q.T                                   # decompositions.cpp:92
    np.linalg.norm(T - rec) / np.linalg.norm(T)      # metrics.cpp:21-28
    t_rec = time.perf_counter() - t0
    scale = N / Ns
    total = (t_qr + t_fwd + t_rec) * scale + t_rsvd + t_svd * p
    detail = {"pixels_sampled": Ns, "pixels": N, "n_linear_scale": scale,
              "qr_s": t_qr * scale, "r_svd_s": t_rsvd, "fwd_s": t_fwd * scale,
              "slice_svd_s": t_svd * p, "slice_svd_each_s": t_svd, "recon_residual_s": t_rec * scale}
    return total, detail
