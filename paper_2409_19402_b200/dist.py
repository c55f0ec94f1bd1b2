"""Multi-GPU tSVDQ with a data-driven basis and multi-GPU star-Q product
(SURVEY §8e), one process per GPU.

tSVDQ (sharded_compress):

The cfg5 pipeline is sharded as follows:

1. Pixels are sharded by lateral j-blocks. Rank r holds A[:, j0:j1, :] as its own
   n1 x nj x n3 tensor. Block boundaries are aligned to the Gram plan's row
   chunks, and the plan depends on (N, n3) only.
2. Each rank computes the partial Grams of its chunks (DMMA SYRK). It reduces them
   locally with the fixed pairwise tree; its chunk group is an aligned power of
   two, so the local result is a subtree. The G subtree roots are all-gathered
   and the same tree is finished on every rank. The Gram, and therefore Q, is
   bitwise identical to the 1-GPU run (verify.cpp:452-455 determinism,
   SURVEY finding 8).
3. The top-p eigensolve is replicated: deterministic, same Q everywhere.
4. The forward transform of the local pixels (A_blk x3 Q^T) runs locally.
5. Â is resharded pixel -> slice by all_to_all_single: each rank gets p/G
   complete slices.
6. The slice SVDs run locally, then the factor stacks are all-gathered.
7. RE from the orthogonal split (Gram trace - ||Ahat||^2 + slice residuals,
   the slice sums all-reduced); below RE^2 = 2e-3 the fused reconstruction
   residual runs over the local pixel block and its two scalars are
   all-reduced instead.

star-Q (sharded_star_q, cfg4): output rows are partitioned. Rank r holds the
row block A[i0:i1, :, :] and the lateral block B[:, j0:j1, :]. It transforms
both locally, all-gathers B^ in slice groups, and runs the facewise GEMMs of a
group into the matching lateral blocks of its C^ rows while the next group is
still in flight. It then applies the inverse transform to its own rows. C has
no reduction, and every element takes the same DMMA accumulation order as the
1-GPU product, so the row blocks are bitwise the 1-GPU C.

Compute goes through a backend object. `DeviceBackend` calls the engine's C-ABI
on CUDA tensors, and collectives use torch.distributed (NCCL on GPUs). The
CPU tests inject a numpy backend over gloo to check the orchestration.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from .projprod import NumericError


def _check(rc):
    if rc:
        raise RuntimeError(_lib.lib().ppc_last_error().decode())


def _fempty(shape, device):
    return torch.empty(tuple(reversed(shape)), dtype=torch.float64,
                       device=device).permute(*reversed(range(len(shape))))


def _p(t):
    return C.c_void_p(t.data_ptr())


class DeviceBackend:
    """The engine's C-ABI on Fortran-laid-out CUDA tensors (loc = PPC_DEVICE)."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.L = _lib.lib()
        _check(self.L.ppc_set_device(self.device.index or 0))
        _check(self.L.ppc_set_stream(C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))

    def gram_plan(self, N, n3):
        c, ch = C.c_int64(), C.c_int64()
        _check(self.L.ppc_gram_plan(N, n3, C.byref(c), C.byref(ch)))
        return c.value, ch.value

    def gram_partials(self, A_blk, rows, n3, chunk, nchunks):
        """Partial Grams of the local chunks; the engine keeps the block's
        7-digit split (when the INT8 path ran on whole 4096-row blocks) for
        mode3_fwd_kept."""
        parts = torch.empty(nchunks * n3 * n3, dtype=torch.float64, device=self.device)
        h = C.c_int64(0)
        bad = C.c_int(0)
        _check(self.L.ppc_gram_partials_keep(_p(A_blk), rows, rows, n3, chunk, nchunks, _p(parts), C.byref(h),
                                             C.byref(bad)))
        self._kept = h.value
        return parts.view(nchunks, n3 * n3), bool(bad.value)

    def release_kept(self):
        h, self._kept = getattr(self, "_kept", 0), 0
        if h:
            _check(self.L.ppc_digits_release(h))

    def mode3_fwd_kept(self, A_blk, n1, nj, n3, Q, p):
        """A_blk x3 Q^T from the digits kept by gram_partials (INT8 tensor
        cores, as the 1-GPU compress); the FP64 DMMA product otherwise."""
        h, self._kept = getattr(self, "_kept", 0), 0
        if h:
            try:
                out = _fempty((n1, nj, p), self.device)
                if self.L.ppc_mode3_forward_digits(h, _p(Q), p, _p(out)) == 0:
                    return out
            finally:
                _check(self.L.ppc_digits_release(h))
        return self.mode3_fwd(A_blk, n1, nj, n3, Q, p)

    def tree_reduce(self, parts):
        """Fixed pairwise tree over the rows of parts (in place); returns row 0."""
        parts = parts.contiguous()
        _check(self.L.ppc_tree_reduce(_p(parts), parts.shape[0], parts.shape[1], 1))
        return parts[0].clone()

    def sym_eig_top(self, G, n3, p):
        Q = _fempty((n3, p), self.device)
        sig = torch.empty(p, dtype=torch.float64, device=self.device)
        _check(self.L.ppc_sym_eig_top(_p(G), n3, p, _p(Q), _p(sig), 1))
        return Q, sig

    # the direct eigensolve split across ranks (ppc_sym_eig_split_*)
    def eig_begin(self, G, n3, p):
        h = C.c_int64(0)
        _check(self.L.ppc_sym_eig_split_begin(_p(G), n3, p, C.byref(h)))
        return h.value or None

    def eig_vectors(self, h, n3, j0, j1):
        Z = _fempty((n3, j1 - j0), self.device)
        _check(self.L.ppc_sym_eig_split_vectors(h, j0, j1, _p(Z)))
        return Z

    def eig_finish(self, h, Zall, n3, j0, j1):
        Q = _fempty((n3, j1 - j0), self.device)
        _check(self.L.ppc_sym_eig_split_finish(h, _p(Zall), j0, j1, _p(Q)))
        return Q

    def eig_release(self, h):
        _check(self.L.ppc_sym_eig_split_release(h))

    def mode3_fwd(self, A_blk, n1, nj, n3, Q, p):
        out = _fempty((n1, nj, p), self.device)
        _check(self.L.ppc_mode3_product(_p(A_blk), n1, nj, n3, _p(Q), p, 1, _p(out), 1))
        return out

    def facewise_into(self, Ah, Bb, Cv):
        """Cv(:, :, s) = Ah(:, :, s) Bb(:, :, s): Ah (a x m x ns) and Bb (m x b x ns)
        Fortran with contiguous slices, Cv a strided (a x b x ns) view into the
        C^ rows. INT8 tensor cores where the 1-GPU star_q's facewise runs there
        (ppc_facewise_strided), else FP64 DMMA."""
        a, m, ns = Ah.shape
        b = Bb.shape[1]
        assert Ah.stride(1) == a and Ah.stride(2) == a * m and Bb.stride(1) == m and Bb.stride(2) == m * b
        _check(self.L.ppc_facewise_strided(_p(Ah), a, m, ns, _p(Bb), b, _p(Cv), Cv.stride(1), Cv.stride(2)))

    def unpack_slices(self, recv, G, ps, nj, n1):
        """recv (G, ps, nj, n1) -> (ps, G nj, n1) whole slices (ppc_reshard_slices)."""
        out = torch.empty((ps, G * nj, n1), dtype=torch.float64, device=self.device)
        _check(self.L.ppc_reshard_slices(_p(recv), G, ps, nj, n1, _p(out)))
        return out

    def mode3_inv(self, Ch, d1, d2, p, Q, n3, scale):
        """(Ch x3 Q) * scale with the 1-GPU star_q's inverse transform
        (ppc_star_inverse: row-wise INT8 digits, so the rank's rows come out
        as in the 1-GPU product) (star_products.cpp:56-58)."""
        out = _fempty((d1, d2, n3), self.device)
        _check(self.L.ppc_star_inverse(_p(Ch), d1 * d2, p, _p(Q), n3, C.c_double(scale), _p(out)))
        return out

    def svd_slices(self, S_loc, n1, n2, ps, k):
        U = _fempty((n1, k, ps), self.device)
        s = _fempty((k, ps), self.device)
        V = _fempty((n2, k, ps), self.device)
        _check(self.L.ppc_svd_batched(_p(S_loc), n1, n2, ps, k, _p(U), _p(s), _p(V), 1))
        return U, s, V

    def gram_trace(self, G, n):
        t = C.c_double()
        _check(self.L.ppc_gram_trace(_p(G), n, C.byref(t), 1))
        return t.value

    def slice_sums(self, S_loc, n1, n2, ps, k, U, s, V):
        sums = (C.c_double * 2)()
        _check(self.L.ppc_slice_residual_sums(_p(S_loc), n1, n2, ps, k, _p(U), _p(s), _p(V), sums, 1))
        return float(sums[0]), float(sums[1])

    def recon_block(self, A_blk, n1, nj, n3, U, S, V, n2, j0, Q, p, k):
        sums = (C.c_double * 2)()
        _check(self.L.ppc_recon_residual_block(_p(A_blk), n1, nj, n3, n1 * nj, _p(U), _p(S), _p(V),
                                               n2, j0, _p(Q), p, k, sums, 1))
        return float(sums[0]), float(sums[1])


@dataclass
class ShardPlan:
    world: int
    rank: int
    n1: int
    n2: int
    n3: int
    p: int
    chunks: int
    chunk: int

    @property
    def cols_per_rank(self):
        return self.n2 // self.world

    @property
    def j0(self):
        return self.rank * self.cols_per_rank

    @property
    def nj(self):
        return self.cols_per_rank

    @property
    def slices_per_rank(self):
        return self.p // self.world

    @property
    def chunks_per_rank(self):
        return self.chunks // self.world


def make_plan(n1, n2, n3, p, world, rank, backend) -> ShardPlan:
    chunks, chunk = backend.gram_plan(n1 * n2, n3)
    if world & (world - 1):
        raise ValueError("world size must be a power of two (pairwise Gram tree)")
    if chunks % world or n2 % world or p % world:
        raise ValueError(f"cannot shard: chunks={chunks}, n2={n2}, p={p} vs world={world}")
    if (n2 // world) * n1 != (chunks // world) * chunk:
        raise ValueError("lateral blocks do not align with the Gram chunks")
    return ShardPlan(world, rank, n1, n2, n3, p, chunks, chunk)


def _tree_finish(roots):
    """Finish the pairwise tree over the G subtree roots (rank order), as the
    engine's tree_reduce does over chunks: width 1, 2, 4, ..."""
    roots = list(roots)
    w = 1
    while w < len(roots):
        for a in range(0, len(roots), 2 * w):
            if a + w < len(roots):
                roots[a] = roots[a] + roots[a + w]
        w *= 2
    return roots[0]


def _gather_cols(X, G, group):
    """all_gather of a Fortran (n, c) column block into Fortran (n, G c),
    columns in rank order (no copy: the gathered buffer is the result)."""
    n, c = X.shape
    out = torch.empty((G * c, n), dtype=X.dtype, device=X.device)
    dist.all_gather_into_tensor(out, X.permute(1, 0).contiguous(), group=group)
    return out.permute(1, 0)


def sharded_eig(Gm, n3, p, rank, G, backend, group=None):
    """Top-p eigenvectors of the (replicated) Gram with the direct solver's
    per-eigenvalue work split across the G ranks (transforms.cpp:97-115:
    U3 = the top eigenvectors of T^T T, sign rule applied)."""
    h = backend.eig_begin(Gm, n3, p) if p % G == 0 else None
    if h is None:
        Q, _ = backend.sym_eig_top(Gm, n3, p)
        return Q
    try:
        j0, j1 = rank * (p // G), (rank + 1) * (p // G)
        Z = backend.eig_vectors(h, n3, j0, j1)
        Zall = _gather_cols(Z, G, group) if G > 1 else Z
        Zall = Zall.permute(1, 0).contiguous().permute(1, 0)
        Ql = backend.eig_finish(h, Zall, n3, j0, j1)
        return _gather_cols(Ql, G, group) if G > 1 else Ql
    finally:
        backend.eig_release(h)


def sharded_compress(A_blk, plan: ShardPlan, k: int, backend, group=None):
    """Runs the sharded pipeline on this rank's lateral block A_blk
    (n1 x nj x n3, Fortran layout). Returns (Q, U, S, V, relative_error) with
    the full factor stacks on every rank."""
    n1, n2, n3, p, nj, G = plan.n1, plan.n2, plan.n3, plan.p, plan.nj, plan.world
    rows = n1 * nj
    # 1-2. partial Grams of the local chunks, local subtree, global finish
    parts, bad = backend.gram_partials(A_blk, rows, n3, plan.chunk, plan.chunks_per_rank)
    # matrix_kernels.cpp:32 on the whole tensor: any rank's NaN/Inf fails all
    flag = torch.tensor([1.0 if bad else 0.0], dtype=torch.float64, device=parts.device)
    if G > 1:
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if float(flag.item()) != 0.0:
        backend.release_kept()
        raise NumericError("svd: input has non-finite entries")
    root = backend.tree_reduce(parts)
    if G > 1:  # the rank subtree roots, finished by the same pairwise tree
        roots = torch.empty((G, root.numel()), dtype=root.dtype, device=root.device)
        dist.all_gather_into_tensor(roots, root.reshape(1, -1), group=group)
        Gm = backend.tree_reduce(roots)
    else:
        Gm = root
    # 3. eigensolve: the tridiagonalization replicated, the eigenvalues and
    #    inverse-iteration vectors of p/G indices per rank, gathered; the
    #    orthonormalization replicated, the back-transformation of p/G columns
    #    per rank, gathered. Q is bitwise the 1-GPU basis for any G.
    Q = sharded_eig(Gm, n3, p, plan.rank, G, backend, group)
    # 4. local forward transform (from the Gram's kept digits when it can)
    Ah = backend.mode3_fwd_kept(A_blk, n1, nj, n3, Q, p)  # (n1, nj, p) Fortran
    # 5. reshard pixel -> slice: chunk for rank s = my block of its slices
    ps = plan.slices_per_rank
    send = Ah.permute(2, 1, 0).contiguous()  # (p, nj, n1) C-order == Fortran (n1, nj, p)
    send = send.view(G, ps * nj * n1)
    recv = torch.empty_like(send)
    if G > 1:
        dist.all_to_all_single(recv, send, group=group)
    else:
        recv.copy_(send)
    # recv[r] = rank r's lateral block (columns j0_r..) of my ps slices
    full = backend.unpack_slices(recv, G, ps, nj, n1) if G > 1 else recv.view(ps, nj, n1)  # [slice][j][i]
    S_loc = full.permute(2, 1, 0)                     # (n1, n2, ps) Fortran view
    # 6. slice SVDs, all-gather the factor stacks
    U, s, V = backend.svd_slices(S_loc, n1, n2, ps, k)
    # slice-space half of the error split, on the local slices (before the gather)
    st, sa2 = backend.slice_sums(S_loc, n1, n2, ps, k, U, s, V)
    Uc = U.permute(2, 1, 0).contiguous()  # (ps, k, n1): no copy, U is Fortran (n1, k, ps)
    sc = s.permute(1, 0).contiguous()     # (ps, k)
    Vc = V.permute(2, 1, 0).contiguous()  # (ps, k, n2)
    if G > 1:  # gathered straight into the (n, k, p) stacks, slices in rank order
        Ug = torch.empty((G * ps,) + tuple(Uc.shape[1:]), dtype=Uc.dtype, device=Uc.device)
        sg = torch.empty((G * ps,) + tuple(sc.shape[1:]), dtype=sc.dtype, device=sc.device)
        Vg = torch.empty((G * ps,) + tuple(Vc.shape[1:]), dtype=Vc.dtype, device=Vc.device)
        dist.all_gather_into_tensor(Ug, Uc, group=group)
        dist.all_gather_into_tensor(sg, sc, group=group)
        dist.all_gather_into_tensor(Vg, Vc, group=group)
        Uc, sc, Vc = Ug, sg, Vg
    Uf, Sf, Vf = Uc.permute(2, 1, 0), sc.permute(1, 0), Vc.permute(2, 1, 0)  # (n1,k,p) (k,p) (n2,k,p)
    # 7. relative error. Q is orthonormal, so ||A - A_k||^2 =
    # (||A||^2 - ||Ahat||^2) + sum_i ||Ahat_i - U_i S_i V_i^T||^2 with ||A||^2 the
    # Gram trace (replicated) and the slice sums all-reduced over the slice
    # shards; when RE^2 < 2e-3 the difference could cancel, so the fused
    # residual runs over the local pixel block instead (engine.cu
    # compress_relative_error; every rank takes the same branch).
    a2 = backend.gram_trace(Gm, n3)
    t = torch.tensor([st, sa2], dtype=torch.float64, device=Ah.device)
    if G > 1:
        dist.all_reduce(t, group=group)
    num = (a2 - float(t[1].item())) + float(t[0].item())
    if a2 > 0.0 and num >= 2e-3 * a2:
        re = (num ** 0.5) / (a2 ** 0.5)
    else:
        sd, sa = backend.recon_block(A_blk, n1, nj, n3, Uf, Sf, Vf, n2, plan.j0, Q, p, k)
        t = torch.tensor([sd, sa], dtype=torch.float64, device=Ah.device)
        if G > 1:
            dist.all_reduce(t, group=group)
        re = float((t[0].sqrt() / t[1].sqrt()).item())
    return Q, Uf, Sf, Vf, re


# ------------------------------------------------------------------ star-Q
@dataclass
class StarPlan:
    world: int
    rank: int
    n1: int
    m: int
    n2: int
    n3: int
    p: int

    @property
    def rows(self):
        return self.n1 // self.world

    @property
    def i0(self):
        return self.rank * self.rows

    @property
    def cols(self):
        return self.n2 // self.world

    @property
    def j0(self):
        return self.rank * self.cols


def make_star_plan(n1, m, n2, n3, p, world, rank) -> StarPlan:
    if n1 % world or n2 % world:
        raise ValueError(f"cannot shard star-Q: n1={n1}, n2={n2} vs world={world}")
    return StarPlan(world, rank, n1, m, n2, n3, p)


def _slice_groups(p, groups):
    groups = max(1, min(groups, p))
    step = -(-p // groups)
    return [(s, min(s + step, p)) for s in range(0, p, step)]


def nccl_gather(group=None, world=1):
    """all_gather of one contiguous tensor, asynchronous: returns a handle
    whose wait() yields the G per-rank tensors."""

    class _H:
        def __init__(self, t):
            self.out = [torch.empty_like(t) for _ in range(world)]
            self.work = dist.all_gather(self.out, t, group=group, async_op=True) if world > 1 else None
            if world == 1:
                self.out[0] = t

        def wait(self):
            if self.work is not None:
                self.work.wait()
            return self.out

    return _H


def sharded_star_q(A_rows, B_cols, Q, plan: StarPlan, backend, scale=1.0, group=None, groups=4,
                   gather=None):
    """star_products.cpp:51-59 on the rank's row block. A_rows is
    (n1/G x m x n3), B_cols is (m x n2/G x n3), both Fortran; Q is n3 x p.
    Returns this rank's rows C[i0:i1, :, :] (n1/G x n2 x n3, Fortran)."""
    Ah = backend.mode3_fwd(A_rows, plan.rows, plan.m, plan.n3, Q, plan.p)   # (rows, m, p)
    Bh = backend.mode3_fwd(B_cols, plan.m, plan.cols, plan.n3, Q, plan.p)   # (m, cols, p)
    return star_finish(Ah, Bh, Q, plan, backend, scale,
                       gather or nccl_gather(group, plan.world), groups)


def star_finish(Ah, Bh, Q, plan: StarPlan, backend, scale, gather, groups=4):
    """All-gather B^ in slice groups (group g+1 in flight while group g's
    facewise GEMMs run), facewise into the C^ rows, inverse transform."""
    G, rows, cols, m, p = plan.world, plan.rows, plan.cols, plan.m, plan.p
    Ch = _fempty((rows, plan.n2, p), Ah.device)
    spans = _slice_groups(p, groups)

    def start(span):
        s0, s1 = span
        send = Bh.permute(2, 1, 0)[s0:s1].contiguous()   # (ns, cols, m) C-order
        return gather(send)

    pending = start(spans[0])
    for g, (s0, s1) in enumerate(spans):
        parts = pending.wait()
        if g + 1 < len(spans):
            pending = start(spans[g + 1])
        for r in range(G):
            Bb = parts[r].permute(2, 1, 0)                  # (m, cols, ns) Fortran
            Cv = Ch[:, r * cols:(r + 1) * cols, s0:s1]
            backend.facewise_into(Ah[:, :, s0:s1], Bb, Cv)
    return backend.mode3_inv(Ch, rows, plan.n2, p, Q, plan.n3, scale)
