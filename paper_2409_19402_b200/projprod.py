"""Python mirror of the reference's `projprod` module (proj/python/bindings.cpp)
on top of the B200 engine's C-ABI (include/ppc.h).

Same names, argument meanings, array layouts and error behaviour as the
reference bindings:
  * tensors are (n1, n2, n3) float64 arrays in the native mode-1-fastest
    layout (bindings.cpp:22-46); factor stacks are (n, k, p) and s is (k, p)
    (bindings.cpp:117-127);
  * shape / bounds / argument / degenerate errors raise ValueError subclasses,
    numeric errors RuntimeError (README.md:135-136, test_smoke.py:99-106).

Arrays may be numpy (host; the engine stages them through HBM) or CUDA torch
tensors laid out Fortran-contiguous (device; zero-copy, stream-ordered). Use
`to_device` / `empty_device` to make such tensors.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = [
    "ShapeError", "BoundsError", "ArgumentError", "DegenerateInputError", "NumericError",
    "FormatError", "EngineError", "Transform", "TsvdqFactors", "mode3_product", "mode_product", "star_q_transpose", "star_q_identity",
    "star_q_rank",
    "facewise_product", "frobenius_norm", "svd", "truncated_svd", "data_dependent_transform",
    "projection_error", "star_q", "star_q_product", "tsvdq", "tsvdq_reconstruct", "tsvdq_error",
    "relative_error", "tsvdq_relative_error", "TsvdqIIFactors", "tsvdq2", "tsvdq2_reconstruct",
    "tsvdq2_error", "read_pt3", "write_pt3", "read_pt3_matrix", "write_pt3_matrix", "pt3_shape",
    "write_tsvdq_factors", "star_m", "star_m_product", "HosvdFactors", "hosvd", "hosvd_reconstruct",
    "MatrixSvdBaseline", "matrix_svd_baseline", "matrix_svd_error", "compress_tsvdq", "tsvdq_sweep", "to_device", "empty_device", "to_host",
    "launch_count", "set_fp64_only", "fp64_only",
]


class ShapeError(ValueError):
    pass


class BoundsError(IndexError, ValueError):
    pass


class ArgumentError(ValueError):
    pass


class DegenerateInputError(ValueError):
    pass


class NumericError(RuntimeError):
    pass


class FormatError(RuntimeError):
    pass


class EngineError(RuntimeError):
    """CUDA runtime failure or no usable B200 (the engine has no CPU path)."""


_ERR = {1: ShapeError, 2: BoundsError, 3: ArgumentError, 4: DegenerateInputError,
        5: NumericError, 6: FormatError, 7: EngineError, 8: EngineError}


def _check(rc: int):
    if rc:
        msg = _lib.lib().ppc_last_error().decode(errors="replace")
        raise _ERR.get(rc, EngineError)(msg)


# ------------------------------------------------------------------ arrays
def _torch():
    import torch
    return torch


def _is_dev(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def _fortran_ok(t) -> bool:
    exp, acc = [], 1
    for s in t.shape:
        exp.append(acc)
        acc *= s
    return all(st == e or sz == 1 for st, e, sz in zip(t.stride(), exp, t.shape))


def empty_device(shape, device="cuda"):
    """Fortran-contiguous float64 CUDA tensor of the given shape."""
    torch = _torch()
    rev = tuple(reversed(tuple(shape)))
    return torch.empty(rev, dtype=torch.float64, device=device).permute(*reversed(range(len(shape))))


def to_device(a, device="cuda"):
    torch = _torch()
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    t = empty_device(a.shape, device)
    t.copy_(torch.from_numpy(a))
    return t


def to_host(x) -> np.ndarray:
    if _is_dev(x):
        return np.asfortranarray(x.cpu().numpy())
    return np.asarray(x)


class _Args:
    """Collects array arguments of one call; all host or all device."""

    def __init__(self, *arrays):
        devs = [_is_dev(a) for a in arrays if a is not None]
        if any(devs) and not all(devs):
            raise ArgumentError("mix of host and device arrays in one call")
        self.device = bool(devs) and all(devs)
        self.loc = _lib.PPC_DEVICE if self.device else _lib.PPC_HOST
        self.keep = []

    def inp(self, a, ndim=None):
        if self.device:
            if a.dtype != _torch().float64:
                raise ArgumentError("device arrays must be float64")
            if not _fortran_ok(a):
                a = a.permute(*reversed(range(a.dim()))).contiguous().permute(*reversed(range(a.dim())))
            self.keep.append(a)
            return a, C.c_void_p(a.data_ptr())
        arr = np.asfortranarray(np.asarray(a, dtype=np.float64))
        if ndim is not None and arr.ndim != ndim:
            raise ShapeError(f"expected a {ndim}-d array, got ndim={arr.ndim}")
        self.keep.append(arr)
        return arr, C.c_void_p(arr.ctypes.data)

    def out(self, shape):
        if self.device:
            t = empty_device(shape)
            self.keep.append(t)
            return t, C.c_void_p(t.data_ptr())
        arr = np.empty(shape, order="F")
        return arr, C.c_void_p(arr.ctypes.data)


def _sync_stream_from_torch():
    """Run the engine on torch's current stream so device arrays are ordered."""
    torch = _torch()
    _check(_lib.lib().ppc_set_stream(C.c_void_p(torch.cuda.current_stream().cuda_stream)))


def _call(args: _Args, fn, *cargs):
    if args.device:
        _sync_stream_from_torch()
    _check(fn(*cargs))


def launch_count(reset: bool = False) -> int:
    return int(_lib.lib().ppc_launch_count(1 if reset else 0))


def set_fp64_only(on: bool = True) -> None:
    """Engine arithmetic (no counterpart in the reference, which is Eigen FP64
    throughout): False (default) runs the large products on the INT8 tensor
    cores as Ozaki FP64 emulation (~1e-14 relative to the operands' scale),
    True runs every product on FP64 DMMA. Process-wide (ppc_set_ozaki)."""
    _check(_lib.lib().ppc_set_ozaki(0 if on else 1))


def fp64_only() -> bool:
    return _lib.lib().ppc_get_ozaki() == 0


# --------------------------------------------------------------- transforms
_KINDS = ("identity", "random", "dct", "haar", "data", "custom")


@dataclass
class Transform:
    """transforms.hpp:23-34: Q (n3 x p, orthonormal columns) + kind/seed/scale."""

    q: np.ndarray
    kind: str = "custom"
    seed: int | None = None
    scale: float = 1.0
    completed_basis: bool = False

    def __init__(self, kind: str, n3: int, p: int, seed: int = 0, data=None):
        # bindings.cpp:73-86 build_transform
        L = _lib.lib()
        if kind not in _KINDS or kind == "custom":
            raise ArgumentError(f"unknown transform '{kind}' (identity|random|dct|haar|data)")
        self.kind, self.scale, self.seed, self.completed_basis = kind, 1.0, None, False
        if kind == "data":
            if data is None:
                raise ArgumentError("transform 'data' needs the data= tensor")
            t = data_dependent_transform(data, p)
            self.q, self.completed_basis = t.q, t.completed_basis
            return
        q = np.empty((int(n3), int(p)), order="F")
        ptr = C.c_void_p(q.ctypes.data)
        if kind == "identity":
            _check(L.ppc_identity_q(n3, p, ptr))
        elif kind == "dct":
            _check(L.ppc_dct_q(n3, p, ptr))
        elif kind == "haar":
            _check(L.ppc_haar_q(n3, p, ptr))
        else:
            _check(L.ppc_random_orthogonal_q(n3, p, C.c_uint64(int(seed)), ptr))
            self.seed = int(seed)
        self.q = q

    @classmethod
    def custom(cls, q, scale: float = 1.0) -> "Transform":
        """transforms.cpp:100-111 custom_transform: Stiefel check, scale != 0."""
        q = np.asfortranarray(np.asarray(q, dtype=np.float64))
        if q.ndim != 2:
            raise ShapeError(f"expected a 2-d array, got ndim={q.ndim}")
        _check(_lib.lib().ppc_check_stiefel(C.c_void_p(q.ctypes.data), q.shape[0], q.shape[1]))
        if scale == 0.0:
            raise ArgumentError("custom_transform: scale must be nonzero")
        t = cls.__new__(cls)
        t.q, t.kind, t.seed, t.scale, t.completed_basis = q, "custom", None, float(scale), False
        return t

    @classmethod
    def _from_q(cls, q, kind="data", completed=False) -> "Transform":
        t = cls.__new__(cls)
        t.q, t.kind, t.seed, t.scale, t.completed_basis = q, kind, None, 1.0, completed
        return t

    @property
    def n3(self) -> int:
        return int(self.q.shape[0])

    @property
    def p(self) -> int:
        return int(self.q.shape[1])


@dataclass
class TsvdqFactors:
    """decompositions.hpp:24-31, exported as bindings.cpp:117-130."""

    u: object   # (n1, k, p)
    s: object   # (k, p)
    v: object   # (n2, k, p)
    transform: Transform
    k: int
    n1: int = field(default=0)
    n2: int = field(default=0)


def _q_of(t, args: _Args):
    q = t.q if isinstance(t, Transform) else t
    if args.device and not _is_dev(q):
        q = to_device(q)
    return args.inp(q, 2)


# ----------------------------------------------------------------- kernels
def mode3_product(a, m):
    """tensor.cpp:139-147: A x_3 M, M is q x n3."""
    args = _Args(a, m if _is_dev(m) else None)
    a_, pa = args.inp(a, 3)
    if args.device and not _is_dev(m):
        m = to_device(m)
    m_, pm = args.inp(m, 2)
    n1, n2, n3 = a_.shape
    if m_.shape[1] != n3:
        raise ShapeError(f"mode3_product: M has {m_.shape[1]} cols, tensor n3={n3}")
    out, po = args.out((n1, n2, m_.shape[0]))
    _call(args, _lib.lib().ppc_mode3_product, pa, n1, n2, n3, pm, m_.shape[0], 0, po, args.loc)
    return out


def mode_product(a, m, mode: int):
    """tensor.cpp:109-137: A x_mode M, M is q x n_mode."""
    if mode == 3:
        return mode3_product(a, m)
    if mode not in (1, 2):
        raise ArgumentError(f"mode_product: mode must be 1, 2 or 3, got {mode}")
    args = _Args(a, m if _is_dev(m) else None)
    a_, pa = args.inp(a, 3)
    if args.device and not _is_dev(m):
        m = to_device(m)
    m_, pm = args.inp(m, 2)
    n1, n2, n3 = a_.shape
    ext = n1 if mode == 1 else n2
    if m_.shape[1] != ext:
        raise ShapeError(f"mode_product({mode}): M has {m_.shape[1]} cols, tensor n{mode}={ext}")
    q = m_.shape[0]
    out, po = args.out((q, n2, n3) if mode == 1 else (n1, q, n3))
    _call(args, _lib.lib().ppc_mode_product, pa, n1, n2, n3, pm, q, mode, po, args.loc)
    return out


def facewise_product(a, b):
    """tensor.cpp:149-156."""
    args = _Args(a, b)
    a_, pa = args.inp(a, 3)
    b_, pb = args.inp(b, 3)
    n1, m, n3 = a_.shape
    if b_.shape[0] != m or b_.shape[2] != n3:
        raise ShapeError(f"facewise_product: {tuple(a_.shape)} vs {tuple(b_.shape)}")
    out, po = args.out((n1, b_.shape[1], n3))
    _call(args, _lib.lib().ppc_facewise_product, pa, n1, m, n3, pb, b_.shape[1], po, args.loc)
    return out


def frobenius_norm(a) -> float:
    args = _Args(a)
    a_, pa = args.inp(a)
    out = C.c_double()
    _call(args, _lib.lib().ppc_frobenius_norm, pa, int(np.prod(a_.shape)), C.byref(out), args.loc)
    return out.value


def truncated_svd(a, k: int):
    """matrix_kernels.cpp:39-46 (batched over a leading stack if a is 3-d:
    a (m, n, batch) -> U (m,k,batch), s (k,batch), V (n,k,batch))."""
    args = _Args(a)
    a_, pa = args.inp(a)
    squeeze = len(a_.shape) == 2
    m, n = a_.shape[0], a_.shape[1]
    batch = 1 if squeeze else a_.shape[2]
    U, pu = args.out((m, k, batch))
    s, ps = args.out((k, batch))
    V, pv = args.out((n, k, batch))
    _call(args, _lib.lib().ppc_svd_batched, pa, m, n, batch, k, pu, ps, pv, args.loc)
    if squeeze:
        return U[:, :, 0], s[:, 0], V[:, :, 0]
    return U, s, V


def svd(a):
    """matrix_kernels.cpp:29-37: thin SVD, descending s, sign rule."""
    shp = a.shape
    return truncated_svd(a, min(shp[0], shp[1]))


def data_dependent_transform(a, p: int) -> Transform:
    """transforms.cpp:97-115 (Gram SYRK + top-p eigensolve on the device)."""
    args = _Args(a)
    a_, pa = args.inp(a, 3)
    n1, n2, n3 = a_.shape
    q, pq = args.out((n3, p))
    comp = C.c_int(0)
    _call(args, _lib.lib().ppc_data_dependent_q, pa, n1, n2, n3, p, pq, None, C.byref(comp), args.loc)
    return Transform._from_q(to_host(q) if args.device else q, "data", bool(comp.value))


def projection_error(a, t) -> float:
    args = _Args(a)
    a_, pa = args.inp(a, 3)
    q_, pq = _q_of(t, args)
    n1, n2, n3 = a_.shape
    if q_.shape[0] != n3:
        raise ShapeError(f"projection_error: transform rows {q_.shape[0]} != tensor n3 {n3}")
    out = C.c_double()
    _call(args, _lib.lib().ppc_projection_error, pa, n1, n2, n3, pq, q_.shape[1], C.byref(out), args.loc)
    return out.value


def star_q_product(a, b, t):
    """star_products.cpp:51-59."""
    args = _Args(a, b)
    a_, pa = args.inp(a, 3)
    b_, pb = args.inp(b, 3)
    q_, pq = _q_of(t, args)
    n1, m, n3 = a_.shape
    if b_.shape[0] != m:
        raise ShapeError(f"star product: inner extents differ ({m} vs {b_.shape[0]})")
    if n3 != q_.shape[0] or b_.shape[2] != q_.shape[0]:
        raise ShapeError("star product: mode-3 extents must match the transform")
    scale = t.scale if isinstance(t, Transform) else 1.0
    out, po = args.out((n1, b_.shape[1], n3))
    _call(args, _lib.lib().ppc_star_q_product, pa, n1, m, n3, pb, b_.shape[1], pq, q_.shape[1],
          C.c_double(scale), po, args.loc)
    return out


star_q = star_q_product


def _host_q(t):
    q = t.q if isinstance(t, Transform) else t
    return to_host(q) if _is_dev(q) else np.asfortranarray(q, dtype=np.float64)


def star_q_transpose(a, t):
    """star_products.cpp:74-85 (bindings.cpp:165-170): transform, transpose
    every slice, transform back. Both mode-3 products run on the GPU."""
    q = _host_q(t)
    a_h = to_host(a) if _is_dev(a) else np.asfortranarray(a, dtype=np.float64)
    if a_h.ndim != 3 or a_h.shape[2] != q.shape[0]:
        raise ShapeError(f"star_q_transpose: mode-3 extent {a_h.shape[2] if a_h.ndim == 3 else '?'} "
                         f"!= transform length {q.shape[0]}")
    ahat = mode3_product(a_h, np.asfortranarray(q.T))
    return mode3_product(np.asfortranarray(ahat.transpose(1, 0, 2)), q)


def star_q_identity(m: int, t):
    """star_products.cpp:61-72 (bindings.cpp:171-176): the m x m x n3 tensor
    whose transform-domain slices are identities, divided by the scale."""
    if m < 1:
        raise ArgumentError("star_q_identity: m must be positive")
    q = _host_q(t)
    ihat = np.zeros((m, m, q.shape[1]), order="F")
    ihat[np.arange(m), np.arange(m), :] = 1.0
    out = mode3_product(ihat, q)
    scale = t.scale if isinstance(t, Transform) else 1.0
    return out if scale == 1.0 else np.asfortranarray(out / scale)


def star_q_rank(a, t, tol_rel: float = 1e-12) -> int:
    """decompositions.cpp:105-114 (bindings.cpp:177-182): the largest numerical
    rank (matrix_kernels.cpp:93-101, s_j > tol_rel * s_0) over the slices of
    A x3 Q^T; the slice SVDs are one batched GPU call."""
    q = _host_q(t)
    a_h = to_host(a) if _is_dev(a) else np.asfortranarray(a, dtype=np.float64)
    if a_h.ndim != 3 or a_h.shape[2] != q.shape[0]:
        raise ShapeError(f"star_q_rank: transform length {q.shape[0]} != tensor n3 "
                         f"{a_h.shape[2] if a_h.ndim == 3 else '?'}")
    ahat = mode3_product(a_h, np.asfortranarray(q.T))
    _, s, _ = svd(ahat)
    s = np.asarray(s).reshape(min(a_h.shape[0], a_h.shape[1]), -1)
    rank = 0
    for i in range(s.shape[1]):
        col = s[:, i]
        r = 0
        while r < col.size and col[r] > tol_rel * col[0]:
            r += 1
        rank = max(rank, r)
    return rank


def star_m_product(a, b, m):
    """star_products.cpp:38-49 (bindings.cpp:151-157 `star_m`)."""
    args = _Args(a, b, m if _is_dev(m) else None)
    a_, pa = args.inp(a, 3)
    b_, pb = args.inp(b, 3)
    if args.device and not _is_dev(m):
        m = to_device(m)
    m_, pm = args.inp(m, 2)
    n1, k, n3 = a_.shape
    if m_.shape[0] != m_.shape[1]:
        raise ShapeError("star_m_product: M must be square")
    if b_.shape[0] != k:
        raise ShapeError(f"star product: inner extents differ ({k} vs {b_.shape[0]})")
    if n3 != m_.shape[0] or b_.shape[2] != m_.shape[0]:
        raise ShapeError("star product: mode-3 extents must match the transform")
    out, po = args.out((n1, b_.shape[1], n3))
    _call(args, _lib.lib().ppc_star_m_product, pa, n1, k, n3, pb, b_.shape[1], pm, po, args.loc)
    return out


star_m = star_m_product


@dataclass
class HosvdFactors:
    """decompositions.hpp:62-67 (bindings.cpp:144-149)."""

    core: object  # (k1, k2, k3)
    u1: object    # (n1, k1)
    u2: object    # (n2, k2)
    u3: object    # (n3, k3)


def hosvd(a, k1: int, k2: int, k3: int) -> HosvdFactors:
    """decompositions.cpp:211-236."""
    args = _Args(a)
    a_, pa = args.inp(a, 3)
    n1, n2, n3 = a_.shape
    if not (1 <= k1 <= n1 and 1 <= k2 <= n2 and 1 <= k3 <= n3):
        raise ArgumentError(f"hosvd: multirank ({k1},{k2},{k3}) outside the tensor extents")
    core, pc = args.out((k1, k2, k3))
    u1, p1 = args.out((n1, k1))
    u2, p2 = args.out((n2, k2))
    u3, p3 = args.out((n3, k3))
    _call(args, _lib.lib().ppc_hosvd, pa, n1, n2, n3, k1, k2, k3, pc, p1, p2, p3, args.loc)
    return HosvdFactors(core, u1, u2, u3)


def hosvd_reconstruct(f: HosvdFactors):
    """decompositions.cpp:238-242."""
    args = _Args(f.core, f.u1, f.u2, f.u3)
    c_, pc = args.inp(f.core, 3)
    u1, p1 = args.inp(f.u1, 2)
    u2, p2 = args.inp(f.u2, 2)
    u3, p3 = args.inp(f.u3, 2)
    k1, k2, k3 = c_.shape
    n1, n2, n3 = u1.shape[0], u2.shape[0], u3.shape[0]
    if (u1.shape[1], u2.shape[1], u3.shape[1]) != (k1, k2, k3):
        raise ShapeError("hosvd_reconstruct: factors do not match the core")
    out, po = args.out((n1, n2, n3))
    _call(args, _lib.lib().ppc_hosvd_reconstruct, pc, k1, k2, k3, p1, n1, p2, n2, p3, n3, po, args.loc)
    return out


@dataclass
class MatrixSvdBaseline:
    """decompositions.hpp:70-74: rank-k SVD of the (n1 n3) x n2 slice stack."""

    u: object  # (n1 n3, k)
    s: object  # (k,)
    v: object  # (n2, k)
    error: float


def matrix_svd_baseline(a, k: int) -> MatrixSvdBaseline:
    """decompositions.cpp:244-255."""
    args = _Args(a)
    a_, pa = args.inp(a, 3)
    n1, n2, n3 = a_.shape
    cap = min(n1 * n3, n2)
    if k < 1 or k > cap:
        raise ArgumentError(f"matrix_svd_baseline: k={k} outside [1,{cap}]")
    U, pu = args.out((n1 * n3, k))
    S, ps = args.out((k,))
    V, pv = args.out((n2, k))
    err = C.c_double()
    _call(args, _lib.lib().ppc_matrix_svd_baseline, pa, n1, n2, n3, k, pu, ps, pv, C.byref(err), args.loc)
    return MatrixSvdBaseline(U, S, V, err.value)


def matrix_svd_error(a, k: int) -> float:
    """bindings.cpp:225-230."""
    return matrix_svd_baseline(a, k).error


def tsvdq(a, t: Transform, k: int) -> TsvdqFactors:
    """decompositions.cpp:62-83."""
    args = _Args(a)
    a_, pa = args.inp(a, 3)
    q_, pq = _q_of(t, args)
    n1, n2, n3 = a_.shape
    if q_.shape[0] != n3:
        raise ShapeError(f"tsvdq: transform length {q_.shape[0]} != tensor n3 {n3}")
    p = q_.shape[1]
    cap = min(n1, n2)
    if k < 1 or k > cap:
        raise ArgumentError(f"tsvdq: k={k} outside [1,{cap}]")
    U, pu = args.out((n1, k, p))
    S, ps = args.out((k, p))
    V, pv = args.out((n2, k, p))
    _call(args, _lib.lib().ppc_tsvdq, pa, n1, n2, n3, pq, p, k, pu, ps, pv, args.loc)
    return TsvdqFactors(U, S, V, t, k, n1, n2)


def _factor_args(f: TsvdqFactors, args: _Args):
    u_, pu = args.inp(f.u, 3)
    s_, ps = args.inp(f.s, 2)
    v_, pv = args.inp(f.v, 3)
    q_, pq = _q_of(f.transform, args)
    return u_, s_, v_, q_, pu, ps, pv, pq


def tsvdq_reconstruct(f: TsvdqFactors):
    """decompositions.cpp:85-94."""
    args = _Args(f.u, f.s, f.v)
    u_, s_, v_, q_, pu, ps, pv, pq = _factor_args(f, args)
    n1, k, p = u_.shape
    n2 = v_.shape[0]
    n3 = q_.shape[0]
    out, po = args.out((n1, n2, n3))
    _call(args, _lib.lib().ppc_tsvdq_reconstruct, pu, ps, pv, pq, n1, n2, n3, p, k, po, args.loc)
    return out


def tsvdq_error(a, f: TsvdqFactors):
    """decompositions.cpp:96-103 -> (total, eckart_young, projection)."""
    args = _Args(a, f.u, f.s, f.v)
    a_, pa = args.inp(a, 3)
    u_, s_, v_, q_, pu, ps, pv, pq = _factor_args(f, args)
    n1, n2, n3 = a_.shape
    if q_.shape[0] != n3:
        raise ShapeError(f"tsvdq_error: transform length {q_.shape[0]} != tensor n3 {n3}")
    k, p = s_.shape
    t, e, pr = C.c_double(), C.c_double(), C.c_double()
    _call(args, _lib.lib().ppc_tsvdq_error, pa, n1, n2, n3, pu, ps, pv, pq, p, k, C.byref(t),
          C.byref(e), C.byref(pr), args.loc)
    return t.value, e.value, pr.value


@dataclass
class TsvdqIIFactors:
    """decompositions.hpp:45-56 (bindings.cpp:132-142). The ragged per-slice
    factors are held padded to r = min(n1, n2) columns: u (n1, r, p), s (r, p),
    v (n2, r, p), zero beyond multirank[i]; uhat(i)/shat(i)/vhat(i) give the
    reference's ragged views."""

    u: object
    s: object
    v: object
    multirank: np.ndarray
    gamma: float
    transform: Transform
    n1: int = field(default=0)
    n2: int = field(default=0)

    @property
    def implicit_rank(self) -> int:
        """decompositions.cpp:116-118: kappa = sum of the multirank."""
        return int(np.sum(self.multirank))

    def uhat(self, i):
        return self.u[:, : int(self.multirank[i]), i]

    def shat(self, i):
        return self.s[: int(self.multirank[i]), i]

    def vhat(self, i):
        return self.v[:, : int(self.multirank[i]), i]


def _i64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def tsvdq2(a, t: Transform, gamma: float) -> TsvdqIIFactors:
    """decompositions.cpp:120-190 (energy-truncated multirank tSVDQ)."""
    args = _Args(a)
    a_, pa = args.inp(a, 3)
    q_, pq = _q_of(t, args)
    n1, n2, n3 = a_.shape
    if q_.shape[0] != n3:
        raise ShapeError(f"tsvdq2: transform length {q_.shape[0]} != tensor n3 {n3}")
    p = q_.shape[1]
    r = min(n1, n2)
    U, pu = args.out((n1, r, p))
    S, ps = args.out((r, p))
    V, pv = args.out((n2, r, p))
    mr = np.zeros(p, dtype=np.int64)
    _call(args, _lib.lib().ppc_tsvdq2, pa, n1, n2, n3, pq, p, C.c_double(gamma), pu, ps, pv,
          _i64p(mr), args.loc)
    return TsvdqIIFactors(U, S, V, mr, float(gamma), t, n1, n2)


def _multirank(f: TsvdqIIFactors, p: int) -> np.ndarray:
    mr = np.ascontiguousarray(f.multirank, dtype=np.int64)
    if mr.shape != (p,):
        raise ShapeError(f"tsvdq2: multirank has {mr.size} entries, transform p={p}")
    return mr


def tsvdq2_reconstruct(f: TsvdqIIFactors):
    """decompositions.cpp:192-201."""
    args = _Args(f.u, f.s, f.v)
    u_, s_, v_, q_, pu, ps, pv, pq = _factor_args(f, args)
    n1, _, p = u_.shape
    n2 = v_.shape[0]
    n3 = q_.shape[0]
    mr = _multirank(f, p)
    out, po = args.out((n1, n2, n3))
    _call(args, _lib.lib().ppc_tsvdq2_reconstruct, pu, ps, pv, pq, n1, n2, n3, p, _i64p(mr), po,
          args.loc)
    return out


def tsvdq2_error(a, f: TsvdqIIFactors):
    """decompositions.cpp:203-209 -> (total, eckart_young, projection)."""
    args = _Args(a, f.u, f.s, f.v)
    a_, pa = args.inp(a, 3)
    u_, s_, v_, q_, pu, ps, pv, pq = _factor_args(f, args)
    n1, n2, n3 = a_.shape
    if q_.shape[0] != n3:
        raise ShapeError(f"tsvdq2_error: transform length {q_.shape[0]} != tensor n3 {n3}")
    if u_.shape[0] != n1 or v_.shape[0] != n2:
        raise ShapeError("tsvdq2_error: factors do not match the tensor")
    p = q_.shape[1]
    mr = _multirank(f, p)
    t, e, pr = C.c_double(), C.c_double(), C.c_double()
    _call(args, _lib.lib().ppc_tsvdq2_error, pa, n1, n2, n3, pu, ps, pv, pq, p, _i64p(mr),
          C.byref(t), C.byref(e), C.byref(pr), args.loc)
    return t.value, e.value, pr.value


# --------------------------------------------------------------------- PT3 I/O
def pt3_shape(path) -> tuple:
    """io.cpp:72-101 header validation: (n1, n2, n3) of a PT3 file."""
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    _check(_lib.lib().ppc_pt3_info(str(path).encode(), C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def read_pt3(path, device=None):
    """io.cpp:72-112 read_pt3. device=None returns a Fortran numpy array;
    device="cuda[:i]" streams the payload straight into a device tensor."""
    n1, n2, n3 = pt3_shape(path)
    if device is None:
        out = np.empty((n1, n2, n3), order="F")
        _check(_lib.lib().ppc_pt3_read(str(path).encode(), C.c_void_p(out.ctypes.data), n1 * n2 * n3,
                                       _lib.PPC_HOST))
        return out
    out = empty_device((n1, n2, n3), device)
    _sync_stream_from_torch()
    _check(_lib.lib().ppc_pt3_read(str(path).encode(), C.c_void_p(out.data_ptr()), n1 * n2 * n3,
                                   _lib.PPC_DEVICE))
    return out


def write_pt3(path, a):
    """io.cpp:52-70 write_pt3 from a host array or a device tensor."""
    if _is_dev(a):
        a_ = a if _fortran_ok(a) else a.permute(*reversed(range(a.dim()))).contiguous().permute(
            *reversed(range(a.dim())))
        shape = tuple(a_.shape) + (1,) * (3 - a_.dim())
        _sync_stream_from_torch()
        _check(_lib.lib().ppc_pt3_write(str(path).encode(), C.c_void_p(a_.data_ptr()), *shape,
                                        _lib.PPC_DEVICE))
        return
    arr = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if arr.ndim not in (2, 3):
        raise ShapeError(f"write_pt3: expected a matrix or an order-3 tensor, got ndim={arr.ndim}")
    shape = arr.shape + (1,) * (3 - arr.ndim)
    _check(_lib.lib().ppc_pt3_write(str(path).encode(), C.c_void_p(arr.ctypes.data), *shape, _lib.PPC_HOST))


def write_pt3_matrix(path, m):
    """io.cpp:114-118: a matrix travels as an n3 = 1 tensor."""
    write_pt3(path, m)


def read_pt3_matrix(path, device=None):
    """io.cpp:120-126: rejects n3 != 1 with FormatError."""
    n1, n2, n3 = pt3_shape(path)
    if n3 != 1:
        raise FormatError(f"{path}: expected a matrix (n3 = 1), got n3 = {n3}")
    t = read_pt3(path, device)
    return t[:, :, 0]


def write_tsvdq_factors(prefix, f: TsvdqFactors):
    """tools/main.cpp:211-222 factor export: <prefix>.U.pt3 (n1,k,p),
    .S.pt3 (k,1,p), .V.pt3 (n2,k,p) and .Q.pt3 (n3,p) as a matrix."""
    write_pt3(f"{prefix}.U.pt3", f.u)
    s = f.s
    if _is_dev(s):
        write_pt3(f"{prefix}.S.pt3", s.unsqueeze(1))
    else:
        write_pt3(f"{prefix}.S.pt3", np.asfortranarray(np.asarray(s))[:, None, :])
    write_pt3(f"{prefix}.V.pt3", f.v)
    q = f.transform.q if isinstance(f.transform, Transform) else f.transform
    write_pt3_matrix(f"{prefix}.Q.pt3", q)


def relative_error(ref, approx) -> float:
    """metrics.cpp:21-28."""
    args = _Args(ref, approx)
    a_, pa = args.inp(ref)
    b_, pb = args.inp(approx)
    if tuple(a_.shape) != tuple(b_.shape):
        raise ShapeError("relative_error: shapes differ")
    out = C.c_double()
    _call(args, _lib.lib().ppc_relative_error, pa, pb, int(np.prod(a_.shape)), C.byref(out), args.loc)
    return out.value


def compress_tsvdq(a, p: int, k: int):
    """tools/main.cpp:186-283 (`compress --method tsvdq --transform data`):
    data-driven Q, tSVDQ factors and the reconstruction's relative error in one
    device pass. Returns (TsvdqFactors, relative_error)."""
    args = _Args(a)
    a_, pa = args.inp(a, 3)
    n1, n2, n3 = a_.shape
    q, pq = args.out((n3, p))
    U, pu = args.out((n1, k, p))
    S, ps = args.out((k, p))
    V, pv = args.out((n2, k, p))
    re = C.c_double()
    _call(args, _lib.lib().ppc_tsvdq_compress, pa, n1, n2, n3, p, k, pq, None, pu, ps, pv,
          C.byref(re), args.loc)
    t = Transform._from_q(to_host(q) if args.device else q, "data")
    return TsvdqFactors(U, S, V, t, k, n1, n2), re.value


def tsvdq_sweep(a, ps, ks, transform=None):
    """tools/main.cpp:299-341 `sweep` (relative error of the rank-k tSVDQ for
    every (p, k)), amortized on the device: one basis (data-driven when
    `transform` is None, else the transform's leading p columns), one slice
    SVD per slice at max k, one fused residual per (p, k).
    Returns an array re[ik, ip]."""
    args = _Args(a)
    a_, pa = args.inp(a, 3)
    n1, n2, n3 = a_.shape
    ps = [int(x) for x in ps]
    ks = [int(x) for x in ks]
    P = (C.c_int64 * len(ps))(*ps)
    K = (C.c_int64 * len(ks))(*ks)
    pq = None
    if transform is not None:
        q = transform.q if isinstance(transform, Transform) else transform
        if args.device and not _is_dev(q):
            q = to_device(q)
        q_, pq = args.inp(q, 2)
    re = np.empty((len(ks), len(ps)), order="F")
    _call(args, _lib.lib().ppc_tsvdq_sweep, pa, n1, n2, n3, P, len(ps), K, len(ks), pq,
          C.c_void_p(re.ctypes.data), args.loc)
    return re


def tsvdq_relative_error(a, f: TsvdqFactors) -> float:
    """relative_error(A, tsvdq_reconstruct(F)) fused (no reconstruction in HBM)."""
    args = _Args(a, f.u, f.s, f.v)
    a_, pa = args.inp(a, 3)
    u_, s_, v_, q_, pu, ps, pv, pq = _factor_args(f, args)
    n1, n2, n3 = a_.shape
    k, p = s_.shape
    out = C.c_double()
    _call(args, _lib.lib().ppc_tsvdq_relative_error, pa, n1, n2, n3, pu, ps, pv, pq, p, k,
          C.byref(out), args.loc)
    return out.value
