"""World-size-2 `gloo` tests of the sharded tSVDQ and star-Q drivers (paper_2409_19402_b200/dist.py)
on CPU, with a numpy stand-in for the engine's per-rank kernels (test-only).

They check the orchestration:
  * the lateral blocks align with the Gram chunks;
  * the pairwise-tree finish over the rank roots reproduces the 1-process
    Gram bitwise;
  * the pixel -> slice reshard (all_to_all_single) assembles the right slices;
  * the factor all-gather and the all-reduced residual give the same Q,
    factors and relative error as the 1-process run.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_19402_b200 import dist as pdist


def _f(t):
    """numpy view of a Fortran-laid-out CPU tensor (no copy when possible)."""
    return np.asfortranarray(t.numpy()) if t.is_contiguous() else t.contiguous().numpy()


def _ft(a):
    a = np.asfortranarray(a)
    return torch.from_numpy(np.ascontiguousarray(a.transpose())).permute(*reversed(range(a.ndim)))


def _sign_rule(U, V):
    for j in range(U.shape[1]):
        i = int(np.argmax(np.abs(U[:, j])))
        if U[i, j] < 0:
            U[:, j] *= -1
            V[:, j] *= -1


class NumpyBackend:
    """Same contract as DeviceBackend, computed with numpy on the host."""

    def gram_plan(self, N, n3):
        # the engine's own plan (host-only C-ABI call, no GPU needed)
        import ctypes as C
        from paper_2409_19402_b200 import _lib
        c, ch = C.c_int64(), C.c_int64()
        assert _lib.lib().ppc_gram_plan(N, n3, C.byref(c), C.byref(ch)) == 0
        return c.value, ch.value

    def gram_partials(self, A_blk, rows, n3, chunk, nchunks):
        T = A_blk.permute(2, 1, 0).contiguous().numpy().reshape(n3, rows).T
        parts = [T[c * chunk:(c + 1) * chunk].T @ T[c * chunk:(c + 1) * chunk] for c in range(nchunks)]
        return torch.from_numpy(np.stack([p.reshape(-1) for p in parts])), not bool(np.isfinite(T).all())

    def release_kept(self):
        pass

    def tree_reduce(self, parts):
        return pdist._tree_finish([parts[i].clone() for i in range(parts.shape[0])])

    def unpack_slices(self, recv, G, ps, nj, n1):
        return recv.view(G, ps, nj, n1).permute(1, 0, 2, 3).reshape(ps, G * nj, n1)

    def eig_begin(self, G, n3, p):
        self._eig = self.sym_eig_top(G, n3, p)[0]
        return 1

    def eig_vectors(self, h, n3, j0, j1):
        return self._eig[:, j0:j1].contiguous()

    def eig_finish(self, h, Zall, n3, j0, j1):
        return Zall[:, j0:j1]

    def eig_release(self, h):
        self._eig = None

    def sym_eig_top(self, G, n3, p):
        w, V = np.linalg.eigh(G.numpy().reshape(n3, n3))
        order = np.argsort(-w, kind="stable")[:p]
        Q = V[:, order].copy()
        _sign_rule(Q, np.zeros_like(Q))
        return _ft(Q), torch.from_numpy(np.sqrt(np.maximum(w[order], 0)))

    def mode3_fwd(self, A_blk, n1, nj, n3, Q, p):
        T = A_blk.permute(2, 1, 0).contiguous().numpy().reshape(n3, n1 * nj).T
        Qn = Q.permute(1, 0).contiguous().numpy().T
        return _ft((T @ Qn).reshape(n1, nj, p, order="F"))

    def mode3_fwd_kept(self, A_blk, n1, nj, n3, Q, p):
        return self.mode3_fwd(A_blk, n1, nj, n3, Q, p)

    def svd_slices(self, S_loc, n1, n2, ps, k):
        S = S_loc.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0)
        U, s, V = np.zeros((n1, k, ps)), np.zeros((k, ps)), np.zeros((n2, k, ps))
        for z in range(ps):
            u, sv, vt = np.linalg.svd(S[:, :, z], full_matrices=False)
            uu, vv = u[:, :k].copy(), vt[:k].T.copy()
            _sign_rule(uu, vv)
            U[:, :, z], s[:, z], V[:, :, z] = uu, sv[:k], vv
        return _ft(U), _ft(s), _ft(V)

    def facewise_into(self, Ah, Bb, Cv):
        a = Ah.numpy()
        b = Bb.numpy()
        c = Cv.numpy()          # strided view sharing Cv's memory
        for s in range(a.shape[2]):
            c[:, :, s] = a[:, :, s] @ b[:, :, s]

    def mode3_inv(self, Ch, d1, d2, p, Q, n3, scale):
        ch = Ch.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0)
        Qn = Q.permute(1, 0).contiguous().numpy().T
        return _ft(scale * np.einsum("ijl,kl->ijk", ch, Qn))

    def gram_trace(self, G, n):
        return float(np.trace(G.numpy().reshape(n, n)))

    def slice_sums(self, S_loc, n1, n2, ps, k, U, s, V):
        S = S_loc.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0)
        Un = U.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0)
        sn = s.permute(1, 0).contiguous().numpy().T
        Vn = V.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0)
        rd = sum(float(np.sum((S[:, :, z] - (Un[:, :, z] * sn[:, z]) @ Vn[:, :, z].T) ** 2)) for z in range(ps))
        return rd, float(np.sum(S ** 2))

    def recon_block(self, A_blk, n1, nj, n3, U, S, V, n2, j0, Q, p, k):
        A = A_blk.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0)
        Un = U.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0)
        Sn = S.permute(1, 0).contiguous().numpy().T
        Vn = V.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0)
        Qn = Q.permute(1, 0).contiguous().numpy().T
        ch = np.stack([(Un[:, :, i] * Sn[:, i]) @ Vn[j0:j0 + nj, :, i].T for i in range(p)], axis=2)
        rec = np.einsum("ijl,kl->ijk", ch, Qn)
        return float(np.sum((A - rec) ** 2)), float(np.sum(A ** 2))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tensor(n1, n2, n3, seed=3, noise=1e-2):
    rng = np.random.default_rng(seed)
    r = 3
    a = np.einsum("ir,jr,kr->ijk", rng.standard_normal((n1, r)), rng.standard_normal((n2, r)),
                  rng.standard_normal((n3, r))) + noise * rng.standard_normal((n1, n2, n3))
    return np.asfortranarray(a)


def _run(rank, world, port, shape, p, k, out_dir, noise=1e-2):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n1, n2, n3 = shape
        a = _tensor(n1, n2, n3, noise=noise)
        be = NumpyBackend()
        plan = pdist.make_plan(n1, n2, n3, p, world, rank, be)
        blk = _ft(a[:, plan.j0:plan.j0 + plan.nj, :])
        Q, U, S, V, re = pdist.sharded_compress(blk, plan, k, be)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), Q=Q.permute(1, 0).contiguous().numpy().T,
                 S=S.permute(1, 0).contiguous().numpy().T, re=re,
                 U=U.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0),
                 V=V.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("noise", [1e-2, 1.0])  # RE^2 below / above 2e-3: direct residual / orthogonal split
def test_sharded_compress_world2_matches_world1(tmp_path, noise):
    shape, p, k = (16, 64, 24), 4, 3
    res = {}
    for world in (1, 2):
        d = tmp_path / f"w{world}"
        d.mkdir()
        mp.spawn(_run, args=(world, _free_port(), shape, p, k, str(d), noise), nprocs=world, join=True)
        res[world] = [np.load(d / f"r{r}.npz") for r in range(world)]
    one = res[1][0]
    for r in res[2]:
        assert np.array_equal(r["Q"], one["Q"])          # bitwise: same Gram tree
        np.testing.assert_allclose(r["S"], one["S"], rtol=1e-12)
        np.testing.assert_allclose(r["U"], one["U"], atol=1e-10)
        np.testing.assert_allclose(r["V"], one["V"], atol=1e-10)
        assert abs(float(r["re"]) - float(one["re"])) <= 1e-13 * float(one["re"])
    # the relative error is the directly measured ||A - tsvdq_reconstruct(F)|| / ||A||
    a = _tensor(*shape, noise=noise)
    Qn = one["Q"]
    ch = np.stack([(one["U"][:, :, i] * one["S"][:, i]) @ one["V"][:, :, i].T for i in range(p)], axis=2)
    rec = np.einsum("ijl,kl->ijk", ch, Qn)
    re_direct = np.linalg.norm(a - rec) / np.linalg.norm(a)
    assert (re_direct ** 2 >= 2e-3) == (noise >= 1.0)
    assert abs(float(one["re"]) - re_direct) <= 1e-12 * re_direct
    # and the 1-process result is the plain (unsharded) pipeline
    T = a.reshape(-1, shape[2], order="F")
    w, Vg = np.linalg.eigh(T.T @ T)
    lam = np.sort(w)[::-1][:p]
    Qn = one["Q"]
    np.testing.assert_allclose(np.sum((T @ Qn) ** 2, axis=0), lam, rtol=1e-10)


def test_plan_rejects_misaligned_shards():
    be = NumpyBackend()
    with pytest.raises(ValueError):
        pdist.make_plan(16, 64, 24, 4, 3, 0, be)   # world not a power of two
    with pytest.raises(ValueError):
        pdist.make_plan(16, 64, 24, 3, 2, 0, be)   # p not divisible


def _star_inputs(n1, m, n2, n3, p):
    rng = np.random.default_rng(11)
    a = np.asfortranarray(rng.standard_normal((n1, m, n3)))
    b = np.asfortranarray(rng.standard_normal((m, n2, n3)))
    q, _ = np.linalg.qr(rng.standard_normal((n3, p)))
    return a, b, np.asfortranarray(q)


def _run_star(rank, world, port, dims, scale, groups, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n1, m, n2, n3, p = dims
        a, b, q = _star_inputs(*dims)
        plan = pdist.make_star_plan(n1, m, n2, n3, p, world, rank)
        A_rows = _ft(a[plan.i0:plan.i0 + plan.rows])
        B_cols = _ft(b[:, plan.j0:plan.j0 + plan.cols])
        Cr = pdist.sharded_star_q(A_rows, B_cols, _ft(q), plan, NumpyBackend(), scale=scale, groups=groups)
        np.save(os.path.join(out_dir, f"c{rank}.npy"), Cr.permute(2, 1, 0).contiguous().numpy().transpose(2, 1, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("groups", [1, 3])
def test_sharded_star_q_world2_matches_product(tmp_path, groups):
    dims, scale = (8, 6, 10, 7, 5), -1.5
    n1, m, n2, n3, p = dims
    a, b, q = _star_inputs(*dims)
    ah = np.einsum("ijk,kl->ijl", a, q)
    bh = np.einsum("ijk,kl->ijl", b, q)
    ch = np.einsum("iml,mjl->ijl", ah, bh)
    want = scale * np.einsum("ijl,kl->ijk", ch, q)  # star_products.cpp:51-59
    for world in (1, 2):
        d = tmp_path / f"w{world}"
        d.mkdir()
        mp.spawn(_run_star, args=(world, _free_port(), dims, scale, groups, str(d)), nprocs=world, join=True)
        got = np.concatenate([np.load(d / f"c{r}.npy") for r in range(world)], axis=0)
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12 * np.abs(want).max())


def test_star_plan_rejects_uneven_rows():
    with pytest.raises(ValueError):
        pdist.make_star_plan(9, 4, 8, 5, 3, 2, 0)
    assert pdist._slice_groups(5, 3) == [(0, 2), (2, 4), (4, 5)]
    assert pdist._slice_groups(2, 8) == [(0, 1), (1, 2)]


def _run_nonfinite(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n1, n2, n3, p = 16, 64, 24, 4
        a = _tensor(n1, n2, n3)
        a[3, 50, 7] = np.nan  # in rank 1's lateral block only
        be = NumpyBackend()
        plan = pdist.make_plan(n1, n2, n3, p, world, rank, be)
        blk = _ft(a[:, plan.j0:plan.j0 + plan.nj, :])
        try:
            pdist.sharded_compress(blk, plan, 3, be)
            msg = "no error"
        except pdist.NumericError as ex:
            msg = "numeric: " + str(ex)
        with open(os.path.join(out_dir, f"e{rank}.txt"), "w") as f:
            f.write(msg)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_compress_nonfinite_fails_every_rank(tmp_path):
    """matrix_kernels.cpp:32 (non-finite SVD input -> numeric_error) on the
    whole tensor: a NaN in one rank's block raises NumericError on both."""
    mp.spawn(_run_nonfinite, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        msg = (tmp_path / f"e{r}.txt").read_text()
        assert msg.startswith("numeric:") and "non-finite" in msg, (r, msg)
