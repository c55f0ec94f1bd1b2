"""ctypes front for the C oracle (oracle/libppo.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py — never by the product
package. Arrays are numpy float64 in Fortran order with the reference's
shapes: tensors (n1, n2, n3), Q (n3, p), factor stacks (n, k, p), s (k, p)
(proj/python/bindings.cpp:22-46,117-127).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libppo.so")
_lib = None

ERRORS = {1: "shape_error", 2: "bounds_error", 3: "argument_error",
          4: "degenerate_input_error", 5: "numeric_error"}


class OracleError(ValueError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        L = C.CDLL(_LIB)
        d, i64, pd = C.c_double, C.c_int64, C.POINTER(C.c_double)
        L.ppo_last_error.restype = C.c_char_p
        L.ppo_frobenius_norm.restype = d
        L.ppo_derive_seed.restype = C.c_uint64
        L.ppo_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ppo_xoshiro_normals.argtypes = [C.c_uint64, pd, i64]
        L.ppo_xoshiro_normals.restype = None
        L.ppo_random_orthogonal_q.argtypes = [i64, i64, C.c_uint64, pd]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _chk(rc):
    if rc:
        raise OracleError(rc, lib().ppo_last_error().decode())


I = C.c_int64


def set_threads(n: int):
    lib().ppo_set_threads(int(n))


def threads() -> int:
    return lib().ppo_threads()


def use_openblas(threads: int = 1) -> bool:
    """Route oracle GEMMs through SciPy's bundled OpenBLAS, standing in for
    Eigen's single-threaded GEMM in the CPU baseline (threads=1, the
    reference's setting); the parity tests use more threads to check
    BASELINE-sized products in seconds."""
    import glob
    import scipy
    libs = glob.glob(os.path.join(os.path.dirname(scipy.__file__), os.pardir,
                                  "scipy.libs", "libscipy_openblas*.so"))
    for path in libs:
        rc = lib().ppo_use_blas(path.encode(), b"scipy_dgemm_",
                                b"scipy_openblas_set_num_threads")
        if rc == 0:
            if threads != 1:
                _chk(lib().ppo_set_blas_threads(int(threads)))
            return True
    return False


def xoshiro_normals(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().ppo_xoshiro_normals(C.c_uint64(seed), _p(out), I(count))
    return out


def derive_seed(seed: int, stream: int) -> int:
    return int(lib().ppo_derive_seed(seed, stream))


def random_tensor(n1, n2, n3, seed):
    """tests/support/common.hpp:45-48: xoshiro256++ normals in buffer order."""
    return xoshiro_normals(seed, n1 * n2 * n3).reshape((n1, n2, n3), order="F")


def random_matrix(m, n, seed):
    return xoshiro_normals(seed, m * n).reshape((m, n), order="F")


def frobenius_norm(a):
    a = _f(a)
    return lib().ppo_frobenius_norm(_p(a), I(a.size))


def mode3_product(a, m):
    a, m = _f(a), _f(m)
    n1, n2, n3 = a.shape
    q = m.shape[0]
    if m.shape[1] != n3:
        raise OracleError(1, "mode3_product: M cols != n3")
    out = np.empty((n1, n2, q), order="F")
    _chk(lib().ppo_mode3_product(_p(a), I(n1), I(n2), I(n3), _p(m), I(q), _p(out)))
    return out


def facewise_product(a, b):
    a, b = _f(a), _f(b)
    n1, m, n3 = a.shape
    if b.shape[0] != m or b.shape[2] != n3:
        raise OracleError(1, "facewise_product: shape mismatch")
    n2 = b.shape[1]
    out = np.empty((n1, n2, n3), order="F")
    _chk(lib().ppo_facewise_product(_p(a), I(n1), I(m), I(n3), _p(b), I(n2), _p(out)))
    return out


def svd(a):
    a = _f(a)
    m, n = a.shape
    r = min(m, n)
    U = np.empty((m, r), order="F")
    s = np.empty(r)
    V = np.empty((n, r), order="F")
    _chk(lib().ppo_svd(_p(a), I(m), I(n), _p(U), _p(s), _p(V)))
    return U, s, V


def orthonormalize(a):
    a = _f(a)
    n, p = a.shape
    Q = np.empty((n, p), order="F")
    _chk(lib().ppo_orthonormalize(_p(a), I(n), I(p), _p(Q)))
    return Q


def dct_q(n3, p):
    Q = np.empty((n3, p), order="F")
    _chk(lib().ppo_dct_q(I(n3), I(p), _p(Q)))
    return Q


def random_orthogonal_q(n3, p, seed):
    Q = np.empty((n3, p), order="F")
    _chk(lib().ppo_random_orthogonal_q(I(n3), I(p), C.c_uint64(seed), _p(Q)))
    return Q


def haar_q(n3, p):
    """transforms.cpp:46-60 (host trivia, restated for the KAT fixtures)."""
    if n3 == 2:
        r = 1 / np.sqrt(2.0)
        H = np.array([[r, r], [r, -r]])
    elif n3 == 4:
        s = np.sqrt(2.0)
        # Eigen's comma initializer fills row by row (transforms.cpp:53-58)
        H = 0.5 * np.array([[1, 1, 1, 1], [1, 1, -1, -1], [s, -s, 0, 0], [0, 0, s, -s]])
    else:
        raise OracleError(3, "haar_transform: n3 must be 2 or 4")
    if p < 1 or p > n3:
        raise OracleError(3, "transform: p outside [1,n3]")
    return np.asfortranarray(H[:, :p])


def data_dependent_q(a, p):
    a = _f(a)
    n1, n2, n3 = a.shape
    Q = np.empty((n3, p), order="F")
    sig = np.zeros(p)
    comp = C.c_int(0)
    _chk(lib().ppo_data_dependent_q(_p(a), I(n1), I(n2), I(n3), I(p), _p(Q), _p(sig),
                                    C.byref(comp)))
    return Q, sig, bool(comp.value)


def projection_error(a, q):
    a, q = _f(a), _f(q)
    n1, n2, n3 = a.shape
    err = C.c_double()
    _chk(lib().ppo_projection_error(_p(a), I(n1), I(n2), I(n3), _p(q), I(q.shape[1]),
                                    C.byref(err)))
    return err.value


def star_q_product(a, b, q, scale=1.0):
    a, b, q = _f(a), _f(b), _f(q)
    n1, m, n3 = a.shape
    n2 = b.shape[1]
    if b.shape[0] != m or b.shape[2] != n3 or q.shape[0] != n3:
        raise OracleError(1, "star product: shape mismatch")
    out = np.empty((n1, n2, n3), order="F")
    _chk(lib().ppo_star_q_product(_p(a), I(n1), I(m), I(n3), _p(b), I(n2), _p(q),
                                  I(q.shape[1]), C.c_double(scale), _p(out)))
    return out


def tsvdq(a, q, k):
    a, q = _f(a), _f(q)
    n1, n2, n3 = a.shape
    p = q.shape[1]
    U = np.empty((n1, k, p), order="F")
    S = np.empty((k, p), order="F")
    V = np.empty((n2, k, p), order="F")
    _chk(lib().ppo_tsvdq(_p(a), I(n1), I(n2), I(n3), _p(q), I(p), I(k), _p(U), _p(S), _p(V)))
    return U, S, V


def slice_spectra(a, q):
    a, q = _f(a), _f(q)
    n1, n2, n3 = a.shape
    p = q.shape[1]
    s = np.empty((min(n1, n2), p), order="F")
    _chk(lib().ppo_slice_spectra(_p(a), I(n1), I(n2), I(n3), _p(q), I(p), _p(s)))
    return s


def tsvdq_reconstruct(U, S, V, q, n3=None):
    U, S, V, q = _f(U), _f(S), _f(V), _f(q)
    n1, k, p = U.shape
    n2 = V.shape[0]
    n3 = q.shape[0]
    out = np.empty((n1, n2, n3), order="F")
    _chk(lib().ppo_tsvdq_reconstruct(_p(U), _p(S), _p(V), _p(q), I(n1), I(n2), I(n3), I(p),
                                     I(k), _p(out)))
    return out


def tsvdq_error(a, U, S, V, q):
    a, U, S, V, q = _f(a), _f(U), _f(S), _f(V), _f(q)
    n1, n2, n3 = a.shape
    k, p = S.shape
    t, e, pr = C.c_double(), C.c_double(), C.c_double()
    _chk(lib().ppo_tsvdq_error(_p(a), I(n1), I(n2), I(n3), _p(U), _p(S), _p(V), _p(q), I(p),
                               I(k), C.byref(t), C.byref(e), C.byref(pr)))
    return t.value, e.value, pr.value


def relative_error(a, ahat):
    a, ahat = _f(a), _f(ahat)
    if a.shape != ahat.shape:
        raise OracleError(1, "relative_error: shapes differ")
    re = C.c_double()
    _chk(lib().ppo_relative_error(_p(a), _p(ahat), I(a.size), C.byref(re)))
    return re.value


def tsvdq2(a, q, gamma):
    """decompositions.cpp:120-209 -> (U (n1,r,p), S (r,p), V (n2,r,p), multirank (p,))
    with r = min(n1, n2) and zero columns beyond each slice's rank."""
    a, q = _f(a), _f(q)
    n1, n2, n3 = a.shape
    p = q.shape[1]
    r = min(n1, n2)
    U = np.empty((n1, r, p), order="F")
    S = np.empty((r, p), order="F")
    V = np.empty((n2, r, p), order="F")
    mr = np.zeros(p, dtype=np.int64)
    _chk(lib().ppo_tsvdq2(_p(a), I(n1), I(n2), I(n3), _p(q), I(p), C.c_double(gamma), _p(U), _p(S),
                          _p(V), mr.ctypes.data_as(C.POINTER(C.c_int64))))
    return U, S, V, mr


def tsvdq2_error(a, U, S, V, q, multirank):
    a, U, S, V, q = _f(a), _f(U), _f(S), _f(V), _f(q)
    n1, n2, n3 = a.shape
    p = q.shape[1]
    mr = np.ascontiguousarray(multirank, dtype=np.int64)
    t, e, pr = C.c_double(), C.c_double(), C.c_double()
    _chk(lib().ppo_tsvdq2_error(_p(a), I(n1), I(n2), I(n3), _p(U), _p(S), _p(V), _p(q), I(p),
                                mr.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(t), C.byref(e),
                                C.byref(pr)))
    return t.value, e.value, pr.value


# ---------------------------------------------------------------- PT3 (io.cpp:52-126)
def pt3_bytes(a) -> bytes:
    """io.cpp:52-70 write_pt3, restated: the exact file bytes for tensor a
    (a matrix is the degenerate n3 = 1 tensor, io.cpp:114-118)."""
    import struct
    a = np.asfortranarray(np.asarray(a, dtype="<f8"))
    shape = a.shape + (1,) * (3 - a.ndim)
    head = b"PT3\0" + struct.pack("<I", 1) + bytes([1, 0, 0, 0]) + struct.pack("<QQQ", *shape)
    return head + a.tobytes(order="F")


def pt3_parse(buf: bytes):
    """io.cpp:72-112 read_pt3, restated; raises ValueError where the reference
    throws format_error."""
    import struct
    if len(buf) < 36:
        raise ValueError("truncated header")
    if buf[:4] != b"PT3\0":
        raise ValueError("bad magic")
    if struct.unpack_from("<I", buf, 4)[0] != 1:
        raise ValueError("unsupported version")
    if buf[8] != 1:
        raise ValueError("unsupported dtype")
    if buf[9] != 0:
        raise ValueError("unsupported field flags")
    n1, n2, n3 = struct.unpack_from("<QQQ", buf, 12)
    if 0 in (n1, n2, n3):
        raise ValueError("zero extent")
    cap = 1 << 59
    if n1 > cap // n2 or n1 * n2 > cap // n3:
        raise ValueError("element count overflows the addressable payload")
    if len(buf) != 36 + 8 * n1 * n2 * n3:
        raise ValueError("payload size mismatch (truncated or trailing bytes)")
    return np.frombuffer(buf, dtype="<f8", offset=36).reshape((n1, n2, n3), order="F")


# ------------------------------------------- star-M and baselines
# numpy/LAPACK restatements (the reference routes these through Eigen's
# JacobiSVD; the SVD here is LAPACK's, with the same sign rule).
def _sign_fix(U, V=None):
    """matrix_kernels.cpp:16-25: largest-|.| entry of each U column (first on
    ties) made nonnegative, V flipped with it."""
    U = U.copy()
    V = None if V is None else V.copy()
    for j in range(U.shape[1]):
        i = int(np.argmax(np.abs(U[:, j])))
        if U[i, j] < 0:
            U[:, j] *= -1
            if V is not None:
                V[:, j] *= -1
    return U, V


def star_m_product(a, b, m):
    """star_products.cpp:38-49."""
    a, b, m = (np.asarray(x, dtype=float) for x in (a, b, m))
    if m.shape[0] != m.shape[1]:
        raise ValueError("star_m_product: M must be square")
    if a.shape[1] != b.shape[0] or a.shape[2] != m.shape[0] or b.shape[2] != m.shape[0]:
        raise ValueError("star product: shape mismatch")
    u, s, vt = np.linalg.svd(m)
    if int(np.sum(s > 1e-12 * s[0])) < m.shape[0]:
        raise ValueError("star_m_product: M is numerically singular")
    minv = vt.T @ np.diag(1.0 / s) @ u.T
    ah = np.einsum("ijk,lk->ijl", a, m)
    bh = np.einsum("ijk,lk->ijl", b, m)
    ch = np.einsum("iml,mjl->ijl", ah, bh)
    return np.asfortranarray(np.einsum("ijk,lk->ijl", ch, minv))


def star_m_by_tubes(a, b, m):
    """tests/support/oracles.hpp:65-80: tube-by-tube summation with an LU solve."""
    a, b, m = (np.asarray(x, dtype=float) for x in (a, b, m))
    out = np.zeros((a.shape[0], b.shape[1], a.shape[2]))
    for j in range(b.shape[1]):
        for i in range(a.shape[0]):
            acc = np.zeros(a.shape[2])
            for l in range(a.shape[1]):
                acc += np.linalg.solve(m, (m @ a[i, l, :]) * (m @ b[l, j, :]))
            out[i, j, :] = acc
    return out


def mode_unfold(a, mode):
    """tensor.cpp:87-107."""
    a = np.asarray(a, dtype=float)
    n1, n2, n3 = a.shape
    if mode == 1:
        return a.reshape(n1, n2 * n3, order="F")
    if mode == 2:
        return np.concatenate([a[:, :, k].T for k in range(n3)], axis=1)
    return a.reshape(n1 * n2, n3, order="F").T


def mode_product(a, m, mode):
    """tensor.cpp:109-137: A x_mode M by index contraction (tests/support/oracles.hpp:82-101)."""
    a = np.asarray(a, dtype=float)
    m = np.asarray(m, dtype=float)
    if mode == 1:
        return np.asfortranarray(np.einsum("qt,tjk->qjk", m, a))
    if mode == 2:
        return np.asfortranarray(np.einsum("qt,itk->iqk", m, a))
    if mode == 3:
        return np.asfortranarray(np.einsum("qt,ijt->ijq", m, a))
    raise ValueError(f"mode_product: mode must be 1, 2 or 3, got {mode}")


def hosvd(a, k1, k2, k3):
    """decompositions.cpp:211-236 -> (core, U1, U2, U3)."""
    a = np.asarray(a, dtype=float)
    if not (1 <= k1 <= a.shape[0] and 1 <= k2 <= a.shape[1] and 1 <= k3 <= a.shape[2]):
        raise ValueError("hosvd: multirank outside the tensor extents")
    fac = []
    for mode, ki in ((1, k1), (2, k2), (3, k3)):
        X = mode_unfold(a, mode)
        # beyond the unfolding's rank: LAPACK's completion of U (full_matrices)
        u, s, vt = np.linalg.svd(X, full_matrices=ki > min(X.shape))
        U, _ = _sign_fix(u[:, :ki], None)
        fac.append(np.asfortranarray(U))
    U1, U2, U3 = fac
    g = np.einsum("ijk,ia->ajk", a, U1)
    g = np.einsum("ajk,jb->abk", g, U2)
    core = np.einsum("abk,kc->abc", g, U3)
    return np.asfortranarray(core), U1, U2, U3


def hosvd_reconstruct(core, U1, U2, U3):
    """decompositions.cpp:238-242."""
    t = np.einsum("abc,ia->ibc", core, U1)
    t = np.einsum("ibc,jb->ijc", t, U2)
    return np.asfortranarray(np.einsum("ijc,kc->ijk", t, U3))


def matrix_svd_baseline(a, k):
    """decompositions.cpp:244-255 -> (U, s, V, error)."""
    a = np.asarray(a, dtype=float)
    n1, n2, n3 = a.shape
    B = np.concatenate([a[:, :, s] for s in range(n3)], axis=0)
    cap = min(B.shape)
    if k < 1 or k > cap:
        raise ValueError("matrix_svd_baseline: k out of range")
    u, s, vt = np.linalg.svd(B, full_matrices=False)
    U, V = _sign_fix(u[:, :k], vt[:k].T)
    err = np.linalg.norm(B - U @ np.diag(s[:k]) @ V.T)
    return U, s[:k].copy(), V, float(err)
