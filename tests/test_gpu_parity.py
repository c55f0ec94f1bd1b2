"""Parity of the CUDA engine (through its C-ABI, via the Python mirror) with
the CPU oracle on the same seeded inputs, plus the reference's known-answer
tests. FP64 tolerances follow BASELINE.json north_star (1e-10 relative on
singular values, reconstructions and relative error) and the reference's own
test tolerances where tighter (1e-12 / 1e-13 for products)."""
import math

import numpy as np
import pytest

from paper_2409_19402_b200 import synth

pytestmark = pytest.mark.gpu
SQ2 = math.sqrt(2.0)


def tube(v):
    return np.asarray(v, dtype=float).reshape(1, 1, -1)


@pytest.fixture(autouse=True)
def _engine_on_torch_stream(engine):
    """Raw C-ABI calls with device pointers are ordered on the engine's current
    stream (loc = PPC_DEVICE is stream-ordered): run it on torch's stream so the
    tensors torch just built are ready, as the Python mirror does per call."""
    import ctypes as C
    import torch
    from paper_2409_19402_b200 import _lib
    assert _lib.lib().ppc_set_stream(C.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    yield


def counterexample():
    a = np.zeros((2, 2, 2))
    a[:, :, 0] = np.eye(2)
    a[:, :, 1] = np.diag([1.0, -1.0])
    return a


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb else 1.0)


# ------------------------------------------------------------- L3 kernels
@pytest.mark.parametrize("shape,q", [((3, 4, 5), 6), ((64, 48, 32), 8), ((37, 29, 61), 13),
                                     ((128, 96, 200), 20), ((256, 128, 256), 64),
                                     ((100, 70, 33), 130), ((16, 8, 7), 1)])
def test_mode3_product_vs_oracle(engine, oracle, shape, q):
    a = oracle.random_tensor(*shape, 13)
    m = oracle.random_matrix(q, shape[2], 14)
    got = engine.mode3_product(a, m)
    want = oracle.mode3_product(a, m)
    assert rel(got, want) <= 1e-13


@pytest.mark.parametrize("shape,q", [((3, 4, 5), 6), ((64, 48, 32), 8), ((37, 29, 61), 13),
                                     ((256, 192, 40), 50), ((16, 8, 7), 1)])
@pytest.mark.parametrize("mode", [1, 2, 3])
def test_mode_product_vs_oracle(engine, oracle, shape, q, mode):
    """tensor.cpp:109-137 (test_tensor.cpp:123-134): modes 1 and 2 (the HOSVD
    baseline's products) and mode 3 against the index-contraction oracle,
    host and device input; the reference's shape and mode errors."""
    import paper_2409_19402_b200 as pp
    a = oracle.random_tensor(*shape, 13)
    m = oracle.random_matrix(q, shape[mode - 1], 14 + mode)
    want = oracle.mode_product(a, m, mode)
    got = engine.mode_product(a, m, mode)
    assert got.shape == want.shape
    assert rel(got, want) <= 1e-13
    got_d = pp.to_host(engine.mode_product(pp.to_device(a), pp.to_device(m), mode))
    assert np.array_equal(got_d, got)
    with pytest.raises(engine.ShapeError):
        engine.mode_product(a, oracle.random_matrix(q, shape[mode - 1] + 1, 3), mode)
    with pytest.raises(engine.ArgumentError):
        engine.mode_product(a, m, 4)


def test_star_q_identity_transpose_rank_reference_cases(engine, oracle):
    """test_star_products.cpp:103-149, test_decompositions.cpp:118-124 and
    tests/python/test_smoke.py:24-44,77-78 through the Python mirror."""
    pp = engine
    a, t = tube([2, 4, 6, 8]), pp.Transform("haar", 4, 2)
    ia = pp.star_q(pp.star_q_identity(1, t), a, t)
    assert np.abs(ia.ravel() - [3, 3, 6, 0]).max() <= 1e-12
    # full transform: a true identity
    A = oracle.random_tensor(3, 4, 4, 9)
    full = pp.Transform("dct", 4, 4)
    assert rel(pp.star_q(pp.star_q_identity(3, full), A, full), A) <= 1e-12
    with pytest.raises(pp.ArgumentError):
        pp.star_q_identity(0, t)
    # transpose rules: (A * B)^T = B^T * A^T; double transpose = the projected part
    A = oracle.random_tensor(3, 2, 5, 10)
    B = oracle.random_tensor(2, 4, 5, 11)
    ctx = pp.Transform("random", 5, 3, seed=13)
    lhs = pp.star_q_transpose(pp.star_q(A, B, ctx), ctx)
    rhs = pp.star_q(pp.star_q_transpose(B, ctx), pp.star_q_transpose(A, ctx), ctx)
    assert lhs.shape == (4, 3, 5)
    assert rel(lhs, rhs) <= 1e-12
    twice = pp.star_q_transpose(pp.star_q_transpose(A, ctx), ctx)
    P = ctx.q @ ctx.q.T
    assert np.linalg.norm(twice - oracle.mode3_product(A, P)) <= 1e-12 * np.linalg.norm(A)
    assert np.linalg.norm(pp.star_q_transpose(np.zeros((2, 3, 5), order="F"), ctx)) == 0.0
    with pytest.raises(pp.ShapeError):
        pp.star_q_transpose(np.zeros((2, 3, 4), order="F"), ctx)
    # star_q_rank
    ce = counterexample()
    assert pp.star_q_rank(ce, pp.Transform("identity", 2, 2)) == 2
    assert pp.star_q_rank(ce, pp.Transform("haar", 2, 1)) == 1
    assert pp.star_q_rank(np.zeros((3, 3, 4), order="F"), pp.Transform("dct", 4, 2)) == 0


@pytest.mark.parametrize("n1,m,n2,p", [(1, 1, 1, 3), (5, 7, 3, 4), (64, 48, 64, 8),
                                       (130, 70, 90, 5), (256, 128, 256, 3)])
def test_facewise_vs_oracle(engine, oracle, n1, m, n2, p):
    a = oracle.random_tensor(n1, m, p, 3)
    b = oracle.random_tensor(m, n2, p, 4)
    assert rel(engine.facewise_product(a, b), oracle.facewise_product(a, b)) <= 1e-13


def test_facewise_tube_kat(engine):
    ab = engine.facewise_product(tube([1, 2, 3]), tube([4, 5, -6])).ravel()
    assert list(ab) == [4.0, 10.0, -18.0]


def test_frobenius_and_relative_error(engine, oracle):
    a = oracle.random_tensor(31, 17, 9, 61)
    assert engine.frobenius_norm(a) == pytest.approx(np.linalg.norm(a), rel=1e-14)
    assert engine.frobenius_norm(counterexample()) == pytest.approx(2.0, rel=1e-15)
    assert engine.frobenius_norm(tube([2, 4, 6, 8])) == pytest.approx(math.sqrt(120.0), rel=1e-15)
    assert engine.relative_error(a, a) == 0.0
    assert engine.relative_error(a, np.zeros_like(a)) == 1.0
    with pytest.raises(engine.DegenerateInputError):
        engine.relative_error(np.zeros_like(a), a)
    with pytest.raises(engine.ShapeError):
        engine.relative_error(a, a[:, :, :3])


# ----------------------------------------------------------- star products
def test_star_q_worked_tube(engine):
    a, b = tube([2, 4, 6, 8]), tube([1, -1, 1, 0])
    t = engine.Transform("haar", 4, 2)
    np.testing.assert_allclose(engine.star_q(a, b, t).ravel(), [3, 3, 3, 0], atol=1e-12)
    h4 = engine.Transform("haar", 4, 4).q
    perp = engine.Transform.custom(h4[:, 2:])
    np.testing.assert_allclose(engine.star_q(a, b, perp).ravel(), [-1, 1, 0, 8], atol=1e-12)


def test_star_q_scale_law(engine):
    rng = np.random.default_rng(8)
    a, b = rng.standard_normal((2, 2, 4)), rng.standard_normal((2, 3, 4))
    unit = engine.Transform("dct", 4, 2)
    base = engine.star_q(a, b, unit)
    for c in (-2.0, 0.5, 3.0):
        got = engine.star_q(a, b, engine.Transform.custom(unit.q, c))
        assert np.linalg.norm(got - c * base) <= 1e-12 * abs(c) * np.linalg.norm(base)


def test_star_q_cfg1_vs_oracle(engine, oracle):
    # BASELINE configs[0]: A 64x48x32 N(0,1) seed 0 (xoshiro, buffer order),
    # Q = random orthogonal (32, 8), A *Q' A^T with A^T the slicewise transpose.
    a = oracle.random_tensor(64, 48, 32, 0)
    at = np.asfortranarray(a.transpose(1, 0, 2))
    q = oracle.random_orthogonal_q(32, 8, 1)
    tq = engine.Transform("random", 32, 8, seed=1)
    assert np.abs(tq.q - q).max() <= 1e-13
    got = engine.star_q(a, at, tq)
    want = oracle.star_q_product(a, at, q)
    assert rel(got, want) <= 1e-12


@pytest.mark.parametrize("n1,m,n2,n3,p", [(128, 64, 96, 64, 16), (96, 80, 112, 40, 40),
                                          (33, 17, 21, 11, 5)])
def test_star_q_vs_oracle(engine, oracle, n1, m, n2, n3, p):
    a = oracle.random_tensor(n1, m, n3, 1)
    b = oracle.random_tensor(m, n2, n3, 2)
    q = oracle.dct_q(n3, p)
    got = engine.star_q(a, b, engine.Transform("dct", n3, p))
    assert rel(got, oracle.star_q_product(a, b, q)) <= 1e-12


def test_star_q_shape_errors(engine):
    t = engine.Transform("dct", 4, 2)
    with pytest.raises(engine.ShapeError):
        engine.star_q(np.ones((2, 3, 4)), np.ones((2, 3, 4)), t)
    with pytest.raises(engine.ShapeError):
        engine.star_q(np.ones((2, 3, 5)), np.ones((3, 3, 5)), t)


# --------------------------------------------------------------- SVD / tSVDQ
def test_svd_contract(engine, oracle):
    a = oracle.random_matrix(7, 5, 21)
    U, s, V = engine.svd(a)
    assert np.all(np.diff(s) <= 0) and s[-1] >= 0
    assert np.linalg.norm(U.T @ U - np.eye(5)) <= 5e-10
    assert np.linalg.norm(V.T @ V - np.eye(5)) <= 5e-10
    assert np.linalg.norm(a - U @ np.diag(s) @ V.T) <= 1e-10 * np.linalg.norm(a)
    Uo, so, Vo = oracle.svd(a)
    np.testing.assert_allclose(s, so, rtol=1e-12)
    np.testing.assert_allclose(U, Uo, atol=1e-10)  # sign rule makes factors comparable
    np.testing.assert_allclose(V, Vo, atol=1e-10)
    _, s, _ = engine.svd(np.array([[SQ2, 0.0], [0.0, 0.0]]))
    assert s[0] == pytest.approx(SQ2, rel=1e-14) and abs(s[1]) <= 1e-14
    aw = oracle.random_matrix(5, 9, 22)  # wide
    U, s, V = engine.svd(aw)
    assert np.linalg.norm(aw - U @ np.diag(s) @ V.T) <= 1e-10 * np.linalg.norm(aw)
    np.testing.assert_allclose(s, oracle.svd(aw)[1], rtol=1e-12)


def test_svd_errors(engine):
    with pytest.raises(engine.ArgumentError):
        engine.truncated_svd(np.ones((3, 2)), 3)
    bad = np.ones((3, 3))
    bad[1, 1] = np.inf
    with pytest.raises(engine.NumericError):
        engine.svd(bad)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1024, 1024, 8), (512, 1024, 8)])
def test_tsvdq_nonfinite_slices_rejected(engine, shape):
    """The svd guard on the transform-domain slices (matrix_kernels.cpp:32):
    tall 1024^2 slices check inside the INT8 slice-Gram split, wide ones
    through the plain scan; either way NumericError, and clean input passes."""
    n1, n2, n3 = shape
    a = synth.cp_tensor_device(n1, n2, n3, rank=5, noise=1e-3, seed=2)
    t = engine.Transform("random", n3, n3, seed=3)
    a[n1 - 7, n2 // 2, 3] = float("nan")
    with pytest.raises(engine.NumericError):
        engine.tsvdq(a, t, 4)
    a[n1 - 7, n2 // 2, 3] = 0.0
    f = engine.tsvdq(a, t, 4)
    assert np.isfinite(engine.to_host(f.s)).all()


def _slice_parity(engine, oracle, a, q, k, s_tol=1e-10, rec_tol=1e-10):
    t = engine.Transform.custom(q)
    f = engine.tsvdq(a, t, k)
    U, S, V = oracle.tsvdq(a, q, k)
    # singular values, relative per value
    ok = S > 1e-13 * S.max()
    assert np.max(np.abs(f.s - S)[ok] / S[ok]) <= s_tol
    # reconstruction, relative to ||A|| (sign/rotation invariant)
    rg = engine.tsvdq_reconstruct(f)
    ro = oracle.tsvdq_reconstruct(U, S, V, q)
    assert rel(rg, ro) <= rec_tol * np.linalg.norm(a) / max(np.linalg.norm(ro), 1e-300)
    # relative error
    reg = engine.relative_error(a, rg)
    reo = oracle.relative_error(a, ro)
    assert abs(reg - reo) <= 1e-10 * max(reo, 1e-300) + 1e-15
    assert abs(engine.tsvdq_relative_error(a, f) - reo) <= 1e-10 * max(reo, 1e-300) + 1e-15
    # factor contracts
    for i in range(q.shape[1]):
        u, v = f.u[:, :, i], f.v[:, :, i]
        assert np.linalg.norm(u.T @ u - np.eye(k)) <= 1e-10 * k
        assert np.linalg.norm(v.T @ v - np.eye(k)) <= 1e-10 * k
        assert np.all(np.diff(f.s[:, i]) <= 0)
    return f


def test_tsvdq_cfg1_vs_oracle(engine, oracle):
    # BASELINE configs[0]: tSVDQ k=4 with the random orthogonal p=8 basis
    a = oracle.random_tensor(64, 48, 32, 0)
    q = oracle.random_orthogonal_q(32, 8, 1)
    f = _slice_parity(engine, oracle, a, q, 4)
    # sign rule -> factors comparable where the gap is clear
    U, S, V = oracle.tsvdq(a, q, 4)
    for i in range(8):
        s = S[:, i]
        for j in range(4):
            gap = min(abs(s[j] - s[j - 1]) if j else np.inf,
                      abs(s[j] - s[j + 1]) if j + 1 < 4 else np.inf) / s[0]
            if gap >= 1e-8:
                assert np.abs(f.u[:, j, i] - U[:, j, i]).max() <= 1e-8
                assert np.abs(f.v[:, j, i] - V[:, j, i]).max() <= 1e-8


def test_tsvdq_error_kats(engine):
    a = counterexample()
    tdd = engine.data_dependent_transform(a, 1)
    tot, ey, pr = engine.tsvdq_error(a, engine.tsvdq(a, tdd, 1))
    assert abs(tot - math.sqrt(3.0)) <= 1e-12
    assert abs(ey - 1.0) <= 1e-12
    assert abs(pr - SQ2) <= 1e-12
    th = engine.Transform("haar", 2, 1)
    f = engine.tsvdq(a, th, 1)
    tot, ey, pr = engine.tsvdq_error(a, f)
    assert abs(tot - SQ2) <= 1e-12 and abs(ey) <= 1e-12 and abs(pr - SQ2) <= 1e-12
    assert abs(engine.relative_error(a, engine.tsvdq_reconstruct(f)) - SQ2 / 2) <= 1e-12


def test_projection_error_kat(engine, oracle):
    assert engine.projection_error(tube([2, 4, 6, 8]), engine.Transform("haar", 4, 2)) == \
        pytest.approx(math.sqrt(66.0), abs=1e-12)
    a = oracle.random_tensor(20, 30, 17, 4)
    q = oracle.dct_q(17, 6)
    assert engine.projection_error(a, engine.Transform("dct", 17, 6)) == pytest.approx(
        oracle.projection_error(a, q), rel=1e-12)


@pytest.mark.parametrize("shape,p", [((67, 63, 37), 1), ((67, 63, 37), 5), ((67, 63, 37), 16), ((67, 63, 37), 17),
                                     ((128, 64, 70), 32), ((129, 65, 130), 20), ((67, 63, 37), 33)])
def test_projection_and_tsvdq_residuals_small_p(engine, oracle, shape, p):
    """The streamed residual kernel (K = p <= 32, tall N >= 4096; p = 33 keeps
    the residual GEMM): projection error and the fused tSVDQ relative error
    against numpy, with ragged row and column tails."""
    a = oracle.random_tensor(*shape, 21)
    t = engine.Transform("random", shape[2], p, seed=3)
    T = a.reshape(-1, shape[2], order="F")
    want = np.linalg.norm(T - (T @ t.q) @ t.q.T)
    assert engine.projection_error(a, t) == pytest.approx(want, rel=1e-12)
    k = 3
    f = engine.tsvdq(a, t, k)
    re = engine.tsvdq_relative_error(a, f)
    rec = oracle.tsvdq_reconstruct(f.u, f.s, f.v, t.q)
    assert re == pytest.approx(np.linalg.norm(a - rec) / np.linalg.norm(a), rel=1e-11)


def test_tsvdq_error_vs_oracle_and_ey_identity(engine, oracle):
    a = oracle.random_tensor(6, 5, 7, 7)
    t = engine.Transform("dct", 7, 4)
    f = engine.tsvdq(a, t, 3)
    tot, ey, pr = engine.tsvdq_error(a, f)
    U, S, V = oracle.tsvdq(a, t.q, 3)
    to, eo, po = oracle.tsvdq_error(a, U, S, V, t.q)
    nrm = np.linalg.norm(a)
    assert abs(tot - to) <= 1e-10 * nrm and abs(ey - eo) <= 1e-10 * nrm and abs(pr - po) <= 1e-10 * nrm
    assert abs(tot ** 2 - (ey ** 2 + pr ** 2)) <= 1e-10 * nrm ** 2
    assert f.u.shape == (6, 3, 4) and f.v.shape == (5, 3, 4) and f.s.shape == (3, 4)


def test_tsvdq_limits(engine, oracle):
    a = oracle.random_tensor(4, 3, 5, 42)
    nrm = np.linalg.norm(a)
    full = engine.Transform("random", 5, 5, seed=9)
    f = engine.tsvdq(a, full, 3)
    assert np.linalg.norm(a - engine.tsvdq_reconstruct(f)) <= 1e-10 * nrm
    tot, ey, pr = engine.tsvdq_error(a, f)
    assert tot <= 1e-10 * nrm and ey <= 1e-10 * nrm and pr <= 1e-10 * nrm
    part = engine.Transform("random", 5, 3, seed=9)
    fp = engine.tsvdq(a, part, 3)
    proj = oracle.mode3_product(a, part.q @ part.q.T)
    assert np.linalg.norm(proj - engine.tsvdq_reconstruct(fp)) <= 1e-10 * nrm
    z = np.zeros((4, 3, 5))
    assert np.linalg.norm(engine.tsvdq_reconstruct(engine.tsvdq(z, part, 2))) == 0.0
    with pytest.raises(engine.ArgumentError):
        engine.tsvdq(a, part, 0)
    with pytest.raises(engine.ArgumentError):
        engine.tsvdq(a, part, 5)


def test_tsvdq_exact_rank(engine, oracle):
    q = oracle.random_orthogonal_q(6, 4, 17)
    hat = np.zeros((5, 4, 4), order="F")
    for s in range(4):
        hat[:, :, s] = oracle.random_matrix(5, 2, 100 + s) @ oracle.random_matrix(4, 2, 200 + s).T
    a = oracle.mode3_product(hat, q)
    f = engine.tsvdq(a, engine.Transform.custom(q), 2)
    tot, ey, pr = engine.tsvdq_error(a, f)
    nrm = np.linalg.norm(a)
    assert abs(tot - pr) <= 1e-10 * nrm and ey <= 1e-10 * nrm and tot <= 1e-10 * nrm


@pytest.mark.parametrize("k", [1, 5, 10, 20])
def test_tsvdq_video_scaled_vs_oracle(engine, oracle, k):
    # cfg2 distribution at 60x80x50 (oracle-sized); shared Q (SURVEY §8c rule 1)
    a = synth.video(60, 80, 50, seed=3)
    q, _, _ = oracle.data_dependent_q(a, 20)
    _slice_parity(engine, oracle, a, q, k)


# --------------------------------------------------------------- data-driven Q
def test_data_q_kats(engine, oracle):
    a = counterexample()
    t = engine.data_dependent_transform(a, 2)
    aq = np.abs(t.q)
    assert np.abs(aq - np.eye(2)).max() <= 1e-12 or np.abs(aq - np.eye(2)[::-1]).max() <= 1e-12
    v = np.array([1 / 3, 2 / 3, 2 / 3])
    b = oracle.random_matrix(2, 2, 5)[:, :, None] * v[None, None, :]
    t1 = engine.data_dependent_transform(b, 1)
    assert min(np.linalg.norm(t1.q[:, 0] - v), np.linalg.norm(t1.q[:, 0] + v)) <= 1e-12
    g = oracle.random_tensor(4, 3, 5, 11)
    assert engine.projection_error(g, engine.data_dependent_transform(g, 5)) <= 1e-10


@pytest.mark.parametrize("shape,p", [((20, 30, 16), 6), ((40, 50, 64), 12), ((3, 2, 9), 8)])
def test_data_q_vs_oracle(engine, oracle, shape, p):
    a = oracle.random_tensor(*shape, 5)
    t = engine.data_dependent_transform(a, p)
    qo, so, comp = oracle.data_dependent_q(a, p)
    assert t.completed_basis == comp
    assert np.abs(t.q.T @ t.q - np.eye(p)).max() <= 1e-12
    n1, n2, n3 = shape
    avail = min(n3, n1 * n2)
    unf = a.reshape(n1 * n2, n3, order="F")
    lam = np.sum((unf @ t.q) ** 2, axis=0)  # captured energy per column = sigma_j^2
    sig2 = so[:min(p, avail)] ** 2
    assert np.max(np.abs(lam[:len(sig2)] - sig2)) <= 1e-12 * sig2[0]
    # projector agreement on the leading block with a clear gap
    pg = t.q[:, :min(p, avail)] @ t.q[:, :min(p, avail)].T
    po = qo[:, :min(p, avail)] @ qo[:, :min(p, avail)].T
    assert np.abs(pg - po).max() <= 1e-9
    # sign rule
    for j in range(min(p, avail)):
        i = int(np.argmax(np.abs(t.q[:, j])))
        assert t.q[i, j] >= 0


def test_data_q_deterministic(engine):
    a = synth.hyperspectral(48, 40, 60, seed=1)
    q1 = engine.data_dependent_transform(a, 12).q
    q2 = engine.data_dependent_transform(a, 12).q
    assert np.array_equal(q1, q2)


def test_hyperspectral_scaled_pipeline(engine, oracle):
    # cfg3 distribution at 64x64x224: data Q p=32 (parity on eigenvalues and
    # captured energy), then tSVDQ k=16 with the shared Q.
    a = synth.hyperspectral(64, 64, 224, seed=2)
    t = engine.data_dependent_transform(a, 32)
    qo, so, _ = oracle.data_dependent_q(a, 32)
    unf = a.reshape(-1, 224, order="F")
    cap_g, cap_o = np.sum((unf @ t.q) ** 2), np.sum((unf @ qo) ** 2)
    assert abs(cap_g - cap_o) <= 1e-12 * cap_o
    _slice_parity(engine, oracle, a, qo, 16)
    # RE with own Q vs oracle with own Q (rule 3)
    f = engine.tsvdq(a, t, 16)
    U, S, V = oracle.tsvdq(a, qo, 16)
    reo = oracle.relative_error(a, oracle.tsvdq_reconstruct(U, S, V, qo))
    assert abs(engine.tsvdq_relative_error(a, f) - reo) <= 1e-10 * reo


# --------------------------------------------------------------- device mode
def test_device_arrays_zero_copy(engine, oracle):
    import torch
    a = oracle.random_tensor(40, 30, 24, 9)
    q = oracle.dct_q(24, 6)
    da = engine.to_device(a)
    t = engine.Transform("dct", 24, 6)
    f = engine.tsvdq(da, t, 5)
    assert isinstance(f.u, torch.Tensor) and f.u.is_cuda
    fh = engine.tsvdq(a, t, 5)
    np.testing.assert_allclose(engine.to_host(f.s), fh.s, rtol=1e-14)
    re_dev = engine.tsvdq_relative_error(da, f)
    assert re_dev == pytest.approx(engine.tsvdq_relative_error(a, fh), rel=1e-13)
    c = engine.star_q(da, engine.to_device(np.asfortranarray(a.transpose(1, 0, 2))), t)
    want = oracle.star_q_product(a, np.asfortranarray(a.transpose(1, 0, 2)), q)
    assert rel(engine.to_host(c), want) <= 1e-12


# ------------------------------------------- large slices (Gram + subspace)
def _numpy_rank_k(a, k):
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    return s, (u[:, :k] * s[:k]) @ vt[:k]


@pytest.mark.parametrize("m,n,k,kind", [(300, 260, 10, "noise"), (256, 256, 16, "spiked"),
                                        (200, 420, 12, "noise"), (512, 384, 32, "lowrank")])
def test_large_slice_svd_vs_lapack(engine, m, n, k, kind):
    rng = np.random.default_rng(m + n + k)
    batch = 3
    a = rng.standard_normal((m, n, batch))
    if kind == "spiked":
        a += 3.0
    if kind == "lowrank":
        a = np.einsum("ir,jr,b->ijb", rng.standard_normal((m, 40)), rng.standard_normal((n, 40)),
                      np.ones(batch)) + 1e-3 * a
    a = np.asfortranarray(a)
    U, s, V = engine.truncated_svd(a, k)
    for z in range(batch):
        sn, ak = _numpy_rank_k(a[:, :, z], k)
        np.testing.assert_allclose(s[:, z], sn[:k], rtol=1e-10)
        rec = (U[:, :, z] * s[:, z]) @ V[:, :, z].T
        assert np.linalg.norm(rec - ak) <= 1e-10 * np.linalg.norm(a[:, :, z])
        assert np.linalg.norm(U[:, :, z].T @ U[:, :, z] - np.eye(k)) <= 1e-10 * k
        assert np.linalg.norm(V[:, :, z].T @ V[:, :, z] - np.eye(k)) <= 1e-10 * k
        for j in range(k):
            i = int(np.argmax(np.abs(U[:, j, z])))
            assert U[i, j, z] >= 0


@pytest.mark.parametrize("m,n,batch", [(512, 520, 16), (301, 333, 5)])
def test_large_slice_svd_direct_batched(engine, m, n, batch):
    """Slice Grams of even order <= ~1536 whose batch fits a few waves of the
    cooperative Householder reduction go to the batched direct eigensolver
    (tridiag_eig.cu; 16 x 512 runs in two waves); odd orders to subspace
    iteration. Both give LAPACK's singular values."""
    import ctypes as C
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(m + batch)
    a = np.asfortranarray(rng.standard_normal((m, n, batch)) + 0.5)
    k = 8
    buf = C.create_string_buffer(1 << 16)
    L.ppc_timing_report(buf, len(buf), 1)  # drop earlier records
    L.ppc_timing_enable(1)
    U, s, V = engine.truncated_svd(a, k)
    L.ppc_timing_report(buf, len(buf), 1)
    L.ppc_timing_enable(0)
    assert ("eig.tridiag" in buf.value.decode()) == (min(m, n) % 2 == 0), buf.value.decode()
    for z in range(batch):
        sn, ak = _numpy_rank_k(a[:, :, z], k)
        np.testing.assert_allclose(s[:, z], sn[:k], rtol=1e-10)
        rec = (U[:, :, z] * s[:, z]) @ V[:, :, z].T
        assert np.linalg.norm(rec - ak) <= 1e-10 * np.linalg.norm(a[:, :, z])


_TRD_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2409_19402_b200 import projprod as P
rng = np.random.default_rng(5)
a = np.asfortranarray(rng.standard_normal((512, 512, 24)) + 0.25)
U, s, V = P.truncated_svd(a, 8)
np.savez(sys.argv[2], U=U, s=s, V=V)
"""


def test_slice_tridiag_l2_copy_matches_shared_memory(tmp_path):
    """The batched Householder reduction with the working copy in L2 (one
    wave, several columns per warp in flight) against the shared-memory
    variant (three waves): same per-lane row order, so the same bits."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    # hybrid: the long-lived (highest) columns of every CTA in shared memory,
    # the rest in L2 (PPC_TRD_HYBRID_KB, off by default)
    for tag, env in (("l2", {}), ("smem", {"PPC_TRD_GMEM": "0"}), ("hybrid", {"PPC_TRD_HYBRID_KB": "200"})):
        f = str(tmp_path / f"{tag}.npz")
        subprocess.run([sys.executable, "-c", _TRD_SCRIPT, root, f], check=True, env={**os.environ, **env},
                       timeout=600)
        out[tag] = np.load(f)
    for key in ("U", "s", "V"):
        assert np.array_equal(out["l2"][key], out["smem"][key]), key
        assert np.array_equal(out["l2"][key], out["hybrid"][key]), key


@pytest.mark.parametrize("m,n", [(300, 260), (301, 261), (260, 300)])
def test_large_slice_svd_direct_zero_and_repeated(engine, m, n):
    """Large-slice path (even order: batched direct eigensolver; odd: subspace
    iteration; wide: A A^T) with a zero slice, a rank-2 slice (k = 6 > rank)
    and a slice of exactly repeated singular values next to a generic one:
    values match LAPACK and U, V are orthonormal for EVERY slice, as the
    reference's JacobiSVD factors are (matrix_kernels.cpp:29-37) -- the
    polish's CholQR2 breaks down on the zero / rank-deficient slices and
    falls back to CGS2 with an orthonormal completion there."""
    rng = np.random.default_rng(5)
    batch, k = 4, 6
    a = np.zeros((m, n, batch))
    a[:, :, 3] = rng.standard_normal((m, 2)) @ rng.standard_normal((2, n))  # rank 2 < k
    a[:, :, 0] = rng.standard_normal((m, n))
    r = min(m, n)
    qu, _ = np.linalg.qr(rng.standard_normal((m, r)))
    qv, _ = np.linalg.qr(rng.standard_normal((n, r)))
    sv = np.concatenate([np.full(10, 3.0), np.linspace(1.0, 0.1, r - 10)])
    a[:, :, 2] = (qu * sv) @ qv.T
    a = np.asfortranarray(a)
    U, s, V = engine.truncated_svd(a, k)
    assert np.isfinite(U).all() and np.isfinite(s).all() and np.isfinite(V).all()
    for z in range(batch):
        sn = np.linalg.svd(a[:, :, z], compute_uv=False)
        np.testing.assert_allclose(s[:, z], sn[:k], rtol=1e-10, atol=1e-12 * max(1.0, sn[0]))
        assert np.linalg.norm(U[:, :, z].T @ U[:, :, z] - np.eye(k)) <= 1e-10 * k, z
        assert np.linalg.norm(V[:, :, z].T @ V[:, :, z] - np.eye(k)) <= 1e-10 * k, z
        for j in range(k):  # sign rule (matrix_kernels.cpp:16-25)
            i = int(np.argmax(np.abs(U[:, j, z])))
            assert U[i, j, z] >= 0, (z, j)
        if z != 2:  # z = 2: the k/k+1 boundary sits inside a repeated cluster
            rec = (U[:, :, z] * s[:, z]) @ V[:, :, z].T
            u_, s_, vt_ = np.linalg.svd(a[:, :, z], full_matrices=False)
            want = (u_[:, :k] * s_[:k]) @ vt_[:k]
            assert np.linalg.norm(rec - want) <= 1e-10 * max(1.0, np.linalg.norm(a[:, :, z])), z


@pytest.mark.parametrize("k", [1, 10, 20])
def test_tsvdq_video_large_slices_vs_oracle(engine, oracle, k):
    # full cfg2 frame size 240x320 (Gram + subspace path), 40 frames
    a = synth.video(240, 320, 40, seed=4)
    q, _, _ = oracle.data_dependent_q(a, 12)
    _slice_parity(engine, oracle, a, q, k)


def test_tsvdq_error_large_slices(engine, oracle):
    a = synth.video(240, 320, 24, seed=5)
    t = engine.Transform("dct", 24, 6)
    f = engine.tsvdq(a, t, 8)
    tot, ey, pr = engine.tsvdq_error(a, f)
    U, S, V = oracle.tsvdq(a, t.q, 8)
    to, eo, po = oracle.tsvdq_error(a, U, S, V, t.q)
    nrm = np.linalg.norm(a)
    assert abs(tot - to) <= 1e-10 * nrm and abs(ey - eo) <= 1e-10 * nrm and abs(pr - po) <= 1e-10 * nrm


def test_data_q_large_n3_vs_oracle(engine, oracle):
    # n3 = 200 > Jacobi limit: Gram + subspace eigensolver for Q (cfg2 p=20)
    a = synth.video(60, 80, 200, seed=6)
    t = engine.data_dependent_transform(a, 20)
    qo, so, _ = oracle.data_dependent_q(a, 20)
    unf = a.reshape(-1, 200, order="F")
    lam = np.sum((unf @ t.q) ** 2, axis=0)
    assert np.max(np.abs(lam - so ** 2)) <= 1e-12 * so[0] ** 2
    assert abs(lam.sum() - (so ** 2).sum()) <= 1e-12 * (so ** 2).sum()
    assert np.abs(t.q.T @ t.q - np.eye(20)).max() <= 1e-12


def test_cp_scaled_pipeline(engine, oracle):
    # cfg5 distribution (rank-50 CP + 1e-3 noise) at 192x176x96, p=64 > rank:
    # noise columns in Q and noise slices (SURVEY finding 8) -> shared-Q parity
    a = synth.cp_tensor(192, 176, 96, rank=50, noise=1e-3, seed=7)
    t = engine.data_dependent_transform(a, 64)
    qo, so, _ = oracle.data_dependent_q(a, 64)
    unf = a.reshape(-1, 96, order="F")
    lam = np.sum((unf @ t.q) ** 2, axis=0)
    assert np.max(np.abs(lam - so ** 2)) <= 1e-12 * so[0] ** 2
    _slice_parity(engine, oracle, a, qo, 16)
    f = engine.tsvdq(a, t, 16)
    U, S, V = oracle.tsvdq(a, qo, 16)
    reo = oracle.relative_error(a, oracle.tsvdq_reconstruct(U, S, V, qo))
    assert abs(engine.tsvdq_relative_error(a, f) - reo) <= 1e-10 * reo


# ------------------------------------------------------------ sharded driver
def test_dist_driver_single_rank_matches_fused(engine):
    # dist.py's per-rank path (DeviceBackend, world=1) against ppc_tsvdq_compress
    import torch
    from paper_2409_19402_b200 import dist as pdist
    a = synth.cp_tensor(96, 128, 64, rank=12, noise=1e-3, seed=11)
    da = engine.to_device(a)
    f, re = engine.compress_tsvdq(da, 16, 6)
    be = pdist.DeviceBackend("cuda:0")
    plan = pdist.make_plan(96, 128, 64, 16, 1, 0, be)
    Q, U, S, V, re2 = pdist.sharded_compress(da, plan, 6, be)
    torch.cuda.synchronize()
    assert np.array_equal(engine.to_host(Q), f.transform.q)  # same Gram tree, same eigensolve
    np.testing.assert_allclose(engine.to_host(S), engine.to_host(f.s), rtol=1e-12)
    assert abs(re2 - re) <= 1e-12 * re


# ------------------------------------------- warp-specialized TMA GEMM path
def _both_paths(fn):
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    outs = []
    for mode in (0, 1):
        assert L.ppc_set_gemm_path(mode) == 0
        try:
            outs.append(fn())
        finally:
            L.ppc_set_gemm_path(0)
    return outs


@pytest.mark.parametrize("shape,q", [((256, 128, 256), 64), ((512, 96, 200), 128), ((300, 100, 64), 32),
                                     ((1024, 64, 96), 20)])
def test_ws_mode3_bitwise_and_vs_numpy(engine, shape, q):
    rng = np.random.default_rng(1)
    a = np.asfortranarray(rng.standard_normal(shape))
    m = np.asfortranarray(rng.standard_normal((q, shape[2])))
    ws, classic = _both_paths(lambda: engine.mode3_product(a, m))
    assert np.array_equal(ws, classic)
    want = np.einsum("ijk,lk->ijl", a, m)
    assert rel(ws, want) <= 1e-13


def test_ws_facewise_starq_bitwise(engine):
    rng = np.random.default_rng(2)
    a = np.asfortranarray(rng.standard_normal((256, 192, 24)))
    b = np.asfortranarray(rng.standard_normal((192, 320, 24)))
    t = engine.Transform("dct", 24, 8)
    f1, f0 = _both_paths(lambda: engine.facewise_product(a, b))
    assert np.array_equal(f1, f0)
    assert rel(f1, np.einsum("imk,mjk->ijk", a, b)) <= 1e-13
    s1, s0 = _both_paths(lambda: engine.star_q(a, b, t))
    assert np.array_equal(s1, s0)


def test_ws_gram_and_residual_bitwise(engine, oracle):
    a = synth.cp_tensor(256, 200, 160, rank=20, noise=1e-3, seed=3)
    q1, q0 = _both_paths(lambda: engine.data_dependent_transform(a, 24).q)
    assert np.array_equal(q1, q0)
    t = engine.Transform.custom(q1)
    f = engine.tsvdq(a, t, 8)
    r1, r0 = _both_paths(lambda: engine.tsvdq_relative_error(a, f))
    assert abs(r1 - r0) <= 1e-15 * r0  # residual partial sums grouped differently
    re = oracle.relative_error(a, oracle.tsvdq_reconstruct(*[engine.to_host(x) for x in (f.u, f.s, f.v)], q1))
    assert abs(r1 - re) <= 1e-12 * re


@pytest.mark.parametrize("n3", [64, 128])
def test_compress_host_streaming_matches_device(engine, oracle, n3):
    # ppc_tsvdq_compress with host buffers streams A in chunk groups and
    # overlaps the upload with the Gram SYRK; results must equal the
    # device-resident call bitwise (same chunks, same tree). n3 = 128: the
    # plan has 16 chunks of 4096 rows on the INT8 path, uploaded in groups of
    # 4, 4, 4, 3 and 1 chunks -- every group takes the plan's path, also the
    # short ones (fewer than 16384 rows).
    a = synth.cp_tensor(256, 256, n3, rank=10, noise=1e-3, seed=9)
    if n3 == 128:
        import ctypes as C
        from paper_2409_19402_b200 import _lib
        c, ch = C.c_int64(), C.c_int64()
        assert _lib.lib().ppc_gram_plan(256 * 256, n3, C.byref(c), C.byref(ch)) == 0
        assert (c.value, ch.value) == (16, 4096)
    fh, reh = engine.compress_tsvdq(a, 16, 8)
    fd, red = engine.compress_tsvdq(engine.to_device(a), 16, 8)
    assert np.array_equal(fh.transform.q, engine.to_host(fd.transform.q))
    assert reh == red
    U, S, V = oracle.tsvdq(a, fh.transform.q, 8)
    reo = oracle.relative_error(a, oracle.tsvdq_reconstruct(U, S, V, fh.transform.q))
    assert abs(reh - reo) <= 1e-10 * reo


# ---------------------------------------------------------- sweep
def test_sweep_vs_oracle(engine, oracle):
    # cfg2 distribution (scaled frames), k in {1, 5, 10, 20} x p in {4, 12, 20}
    a = synth.video(60, 80, 50, seed=12)
    ps, ks = [4, 12, 20], [1, 5, 10, 20]
    re = engine.tsvdq_sweep(a, ps, ks)
    qmax, _, _ = oracle.data_dependent_q(a, 20)
    for ip, p in enumerate(ps):
        q = qmax[:, :p]  # data_dependent_transform(A, p) = U3(:, 1:p)
        for ik, k in enumerate(ks):
            U, S, V = oracle.tsvdq(a, q, k)
            want = oracle.relative_error(a, oracle.tsvdq_reconstruct(U, S, V, q))
            assert abs(re[ik, ip] - want) <= 1e-10 * want, (p, k)
    # with a given basis; and the reference's grid checks
    t = engine.Transform("dct", 50, 20)
    re2 = engine.tsvdq_sweep(a, [20], [10], t)
    f = engine.tsvdq(a, t, 10)
    assert abs(re2[0, 0] - engine.tsvdq_relative_error(a, f)) <= 1e-12 * re2[0, 0]
    with pytest.raises(engine.ArgumentError):
        engine.tsvdq_sweep(a, [51], [1])
    with pytest.raises(engine.ArgumentError):
        engine.tsvdq_sweep(a, [4], [61])


def test_sweep_small_errors_direct_residual(engine, oracle):
    """RE^2 below 2e-3 of ||A||^2: the sweep measures the residual directly
    against A instead of through the orthogonal split (no cancellation)."""
    rng = np.random.default_rng(21)
    a = np.einsum("ir,jr,kr->ijk", rng.standard_normal((30, 3)), rng.standard_normal((20, 3)),
                  rng.standard_normal((16, 3)))
    a = np.asfortranarray(a + 1e-5 * rng.standard_normal(a.shape))
    # a fixed basis (a data-driven one's noise directions are not determined
    # to 1e-10): p = 16 keeps all of mode 3 (RE ~ 1e-5, direct residual),
    # p = 8 drops half of it (RE ~ 0.5, orthogonal split)
    ps, ks = [8, 16], [3, 5]
    re = engine.tsvdq_sweep(a, ps, ks, engine.Transform("dct", 16, 16))
    qmax = oracle.dct_q(16, 16)
    for ip, p in enumerate(ps):
        for ik, k in enumerate(ks):
            q = qmax[:, :p]
            U, S, V = oracle.tsvdq(a, q, k)
            want = oracle.relative_error(a, oracle.tsvdq_reconstruct(U, S, V, q))
            assert (want < 1e-3) == (p == 16)
            assert abs(re[ik, ip] - want) <= 1e-10 * want, (p, k, re[ik, ip], want)


def test_sweep_large_slices(engine, oracle):
    a = synth.video(240, 320, 30, seed=13)
    ps, ks = [8, 16], [2, 12]
    re = engine.tsvdq_sweep(a, ps, ks)
    qmax, _, _ = oracle.data_dependent_q(a, 16)
    for ip, p in enumerate(ps):
        for ik, k in enumerate(ks):
            q = qmax[:, :p]
            U, S, V = oracle.tsvdq(a, q, k)
            want = oracle.relative_error(a, oracle.tsvdq_reconstruct(U, S, V, q))
            assert abs(re[ik, ip] - want) <= 1e-10 * want


# ------------------------------------------------------------------ tsvdq2
def _tsvdq2_parity(engine, oracle, a, q, gamma):
    f = engine.tsvdq2(a, engine.Transform.custom(q) if not isinstance(q, engine.Transform) else q, gamma)
    qq = q.q if isinstance(q, engine.Transform) else q
    U, S, V, mr = oracle.tsvdq2(a, qq, gamma)
    assert list(f.multirank) == list(mr)
    assert f.implicit_rank == int(mr.sum())
    r = min(a.shape[0], a.shape[1])
    assert f.u.shape == (a.shape[0], r, qq.shape[1]) and f.s.shape == (r, qq.shape[1])
    smax = max(S.max(), 1e-300)
    assert np.abs(f.s - S).max() <= 1e-10 * smax
    nrm = np.linalg.norm(a)
    rec = engine.tsvdq2_reconstruct(f)
    assert np.linalg.norm(rec - oracle.tsvdq_reconstruct(U, S, V, qq, a.shape[2])) <= 1e-10 * nrm
    got = engine.tsvdq2_error(a, f)
    want = oracle.tsvdq2_error(a, U, S, V, qq, mr)
    for g, w in zip(got, want):
        assert abs(g - w) <= 1e-10 * nrm
    for i in range(qq.shape[1]):  # kept columns orthonormal, dropped ones zero
        k = int(f.multirank[i])
        u = f.u[:, :k, i]
        assert np.linalg.norm(u.T @ u - np.eye(k)) <= 1e-10 * max(k, 1)
        assert not f.u[:, k:, i].any() and not f.s[k:, i].any() and not f.v[:, k:, i].any()
    return f


def test_tsvdq2_reference_cases(engine, oracle):
    # tests/test_decompositions.cpp:126-146
    a = oracle.random_tensor(4, 5, 6, 44)
    t = engine.Transform("dct", 6, 4)
    f = _tsvdq2_parity(engine, oracle, a, t, 1.0)
    tot, ey, _ = engine.tsvdq2_error(a, f)
    assert abs(tot - engine.projection_error(a, t)) <= 1e-10 * np.linalg.norm(a)
    assert ey <= 1e-10 * np.linalg.norm(a)
    for g in (0.0, 1.5):
        with pytest.raises(engine.ArgumentError):
            engine.tsvdq2(a, t, g)
    # :148-160 tie-break
    c = counterexample()
    f = engine.tsvdq2(c, engine.Transform("identity", 2, 2), 0.5)
    assert list(f.multirank) == [2, 0] and f.implicit_rank == 2
    assert abs(engine.tsvdq2_error(c, f)[0] ** 2 - 2.0) <= 1e-12
    # :179-188 full transform lossless
    a = oracle.random_tensor(3, 4, 4, 46)
    tot, ey, pr = engine.tsvdq2_error(a, engine.tsvdq2(a, engine.Transform("dct", 4, 4), 1.0))
    assert max(tot, ey, pr) <= 1e-10 * np.linalg.norm(a)
    # :190-205 error decomposition
    for i in range(10):
        a = oracle.random_tensor(4, 3, 5, 470 + i)
        f = engine.tsvdq2(a, engine.Transform("random", 5, 3, seed=100 + i), 0.8)
        tot, ey, pr = engine.tsvdq2_error(a, f)
        assert abs(tot ** 2 - (ey ** 2 + pr ** 2)) <= 1e-10 * tot ** 2
        assert abs(tot - np.linalg.norm(a - engine.tsvdq2_reconstruct(f))) <= 1e-10 * np.linalg.norm(a)


def test_tsvdq2_exact_rank_matches_tsvdq(engine, oracle):
    # tests/test_decompositions.cpp:162-177; verify.cpp:833-848
    q = oracle.dct_q(5, 3)
    hat = np.zeros((4, 4, 3), order="F")
    for s in range(3):
        hat[:, :, s] = oracle.random_matrix(4, 2, 300 + s) @ oracle.random_matrix(4, 2, 400 + s).T
    a = oracle.mode3_product(hat, q)
    t = engine.Transform.custom(q)
    f2 = engine.tsvdq2(a, t, 1.0)
    assert list(f2.multirank) == [2, 2, 2]
    f1 = engine.tsvdq(a, t, 2)
    nrm = np.linalg.norm(a)
    assert np.linalg.norm(engine.tsvdq2_reconstruct(f2) - engine.tsvdq_reconstruct(f1)) <= 1e-12 * nrm
    assert abs(engine.tsvdq2_error(a, f2)[0] - engine.tsvdq_error(a, f1)[0]) <= 1e-12 * nrm


@pytest.mark.parametrize("shape,p,gamma", [((6, 5, 7), 4, 0.9), ((64, 48, 32), 8, 0.5),
                                           ((37, 29, 20), 20, 0.99), ((30, 40, 12), 5, 0.3),
                                           ((200, 180, 6), 3, 0.7)])
def test_tsvdq2_vs_oracle(engine, oracle, shape, p, gamma):
    a = oracle.random_tensor(*shape, 7 + p)
    q = oracle.random_orthogonal_q(shape[2], p, 3)
    _tsvdq2_parity(engine, oracle, a, q, gamma)


def test_tsvdq2_video_and_dominance(engine, oracle):
    # verify.cpp:796-822: gamma set to the energy tsvdq keeps at k -> tsvdq2 is
    # no worse and keeps at most k*p triplets
    a = synth.video(60, 80, 50, seed=3)
    q, _, _ = oracle.data_dependent_q(a, 20)
    t = engine.Transform.custom(q)
    ahat2 = np.linalg.norm(oracle.mode3_product(a, q.T)) ** 2
    for k in (1, 5, 10):
        es = engine.tsvdq_error(a, engine.tsvdq(a, t, k))
        gamma = min(1.0, max((ahat2 - es[1] ** 2) / ahat2, 1e-300)) * (1 - 1e-12)
        f2 = _tsvdq2_parity(engine, oracle, a, q, gamma)
        assert f2.implicit_rank <= k * 20
        assert engine.tsvdq2_error(a, f2)[0] <= es[0] * (1 + 1e-12)


def test_tsvdq2_device_arrays_and_zero(engine, oracle):
    import torch
    a = oracle.random_tensor(24, 20, 16, 5)
    q = oracle.dct_q(16, 6)
    t = engine.Transform.custom(q)
    fh = engine.tsvdq2(a, t, 0.75)
    fd = engine.tsvdq2(engine.to_device(a), t, 0.75)
    assert isinstance(fd.u, torch.Tensor) and fd.u.is_cuda
    assert list(fd.multirank) == list(fh.multirank)
    assert np.array_equal(engine.to_host(fd.s), fh.s)
    rd = engine.to_host(engine.tsvdq2_reconstruct(fd))
    assert np.array_equal(rd, engine.tsvdq2_reconstruct(fh))
    assert engine.tsvdq2_error(engine.to_device(a), fd) == engine.tsvdq2_error(a, fh)
    z = np.zeros((5, 4, 6))
    fz = engine.tsvdq2(z, engine.Transform("dct", 6, 3), 1.0)
    assert list(fz.multirank) == [0, 0, 0]
    assert not engine.tsvdq2_reconstruct(fz).any()


# ------------------------------------------------------- sharded star-Q (cfg4 §8e)
CFG4 = (1024, 512, 1024, 256, 64)


@pytest.mark.parametrize("world,groups,dims", [(1, 4, None), (2, 3, None), (4, 1, None), (2, 4, CFG4),
                                              (8, 4, CFG4)])
def test_sharded_star_q_rows_bitwise(engine, world, groups, dims):
    """Every rank's row block of the sharded product equals the 1-GPU
    ppc_star_q_product rows bitwise. Ranks run one after another on one GPU:
    phase 1 (local transforms) for all ranks, then each rank's finish with a
    gather that hands back the precomputed B^ groups (no cross-rank waits).
    At the cfg4 shape both run the facewise on the INT8 tensor cores (the
    rank's 128-row blocks and B's columns split exactly as in the 1-GPU
    product)."""
    import torch
    from paper_2409_19402_b200 import dist as pdist
    n1, m, n2, n3, p = dims or (96, 80, 128, 40, 12)
    scale = 0.75
    A = synth.gaussian_device(n1, m, n3, 5, 1)
    B = synth.gaussian_device(m, n2, n3, 5, 2)
    Q = engine.to_device(engine.Transform("dct", n3, p).q)
    want = engine.to_host(engine.star_q_product(A, B, engine.Transform.custom(engine.to_host(Q), scale)))
    be = pdist.DeviceBackend("cuda:0")
    plans = [pdist.make_star_plan(n1, m, n2, n3, p, world, r) for r in range(world)]

    def rows_of(x, pl):
        return x[pl.i0:pl.i0 + pl.rows].permute(2, 1, 0).contiguous().permute(2, 1, 0)

    def cols_of(x, pl):
        return x[:, pl.j0:pl.j0 + pl.cols].permute(2, 1, 0).contiguous().permute(2, 1, 0)

    Bh = [be.mode3_fwd(cols_of(B, pl), m, pl.cols, n3, Q, p) for pl in plans]

    class Pre:
        """Hands back the G ranks' B^ blocks of the next slice group."""

        def __init__(self, spans):
            self.spans = iter(spans)

        def __call__(self, send):
            s0, s1 = next(self.spans)
            assert send.shape[0] == s1 - s0
            parts = [Bh[q].permute(2, 1, 0)[s0:s1].contiguous() for q in range(world)]

            class H:
                def wait(self):
                    return parts
            return H()

    for r, pl in enumerate(plans):
        Ah = be.mode3_fwd(rows_of(A, pl), pl.rows, m, n3, Q, p)
        gather = Pre(pdist._slice_groups(p, groups))
        Cr = pdist.star_finish(Ah, Bh[r], Q, pl, be, scale, gather, groups)
        torch.cuda.synchronize()
        got = engine.to_host(Cr)
        assert np.array_equal(got, want[pl.i0:pl.i0 + pl.rows]), f"rank {r}"


# ------------------------------------------------------------ PT3 device streaming
def test_pt3_device_streaming_round_trip(engine, tmp_path):
    """A file larger than one 64 MiB staging chunk streams into and out of
    device memory bit-exactly (two alternating pinned buffers)."""
    import torch
    a = synth.gaussian_device(512, 400, 50, 3, 1)          # 81.9 MB payload
    f = tmp_path / "big.pt3"
    engine.write_pt3(f, a)                                  # device -> file
    h = engine.read_pt3(f)                                  # file -> host
    assert np.array_equal(h, engine.to_host(a))
    d = engine.read_pt3(f, device="cuda")                   # file -> device
    assert d.is_cuda and torch.equal(d, a)


def test_pt3_compress_chain(engine, oracle, tmp_path):
    """tools/main.cpp:186-222 compress chain: read_pt3 -> data transform ->
    tsvdq -> factor export, on the device; exported factors read back equal."""
    a = synth.video(60, 80, 50, seed=3)
    f = tmp_path / "video.pt3"
    engine.write_pt3(f, a)
    ad = engine.read_pt3(f, device="cuda")
    t = engine.data_dependent_transform(ad, 20)
    fac = engine.tsvdq(ad, t, 5)
    pre = str(tmp_path / "fac")
    engine.write_tsvdq_factors(pre, fac)
    assert np.array_equal(engine.read_pt3(pre + ".U.pt3"), engine.to_host(fac.u))
    assert np.array_equal(engine.read_pt3(pre + ".S.pt3")[:, 0, :], engine.to_host(fac.s))
    assert np.array_equal(engine.read_pt3(pre + ".V.pt3"), engine.to_host(fac.v))
    assert np.array_equal(engine.read_pt3_matrix(pre + ".Q.pt3"), engine.to_host(t.q))
    # and the host path gives the same factors
    fh = engine.tsvdq(a, engine.Transform.custom(engine.to_host(t.q)), 5)
    assert np.abs(fh.s - engine.to_host(fac.s)).max() <= 1e-12 * fh.s.max()


# ---------------------------------------------- star-M and baselines
def test_star_m_kats(engine, oracle):
    # tests/test_star_products.cpp:34-68
    a, b = tube([2, 4, 6, 8]), tube([1, -1, 1, 0])
    h4 = engine.Transform("haar", 4, 4).q
    np.testing.assert_allclose(engine.star_m_product(a, b, h4.T).ravel(), [2, 4, 3, 8], atol=1e-12)
    np.testing.assert_allclose(engine.star_m_product(tube([1, 2, 3]), tube([4, -5, 0.5]), np.eye(3)).ravel(),
                               [4, -10, 1.5], atol=1e-14)
    A = oracle.random_tensor(2, 3, 4, 31)
    B = oracle.random_tensor(3, 2, 4, 32)
    M = oracle.random_matrix(4, 4, 33)
    fast = engine.star_m_product(A, B, M)
    assert np.linalg.norm(fast - oracle.star_m_by_tubes(A, B, M)) <= 1e-12 * np.linalg.norm(fast)
    sing = np.zeros((2, 2))
    sing[0, 0] = 1.0
    with pytest.raises(engine.DegenerateInputError):
        engine.star_m_product(tube([1, 2]), tube([1, 2]), sing)
    with pytest.raises(engine.ShapeError):
        engine.star_m_product(tube([1, 2]), tube([1, 2, 3]), np.eye(2))
    wide = np.zeros((1, 2, 2))
    with pytest.raises(engine.ShapeError):
        engine.star_m_product(wide, wide, np.eye(2))
    # test_star_products.cpp:80-88: star_q with p = n3 is star_m with M = Q^T
    A = oracle.random_tensor(3, 4, 6, 34)
    B = oracle.random_tensor(4, 2, 6, 35)
    t = engine.Transform("random", 6, 6, seed=36)
    sq = engine.star_q_product(A, B, t)
    sm = engine.star_m_product(A, B, t.q.T)
    assert np.linalg.norm(sq - sm) <= 1e-12 * np.linalg.norm(sq)


@pytest.mark.parametrize("n1,m,n2,n3", [(37, 29, 41, 24), (64, 96, 80, 200)])
def test_star_m_vs_oracle(engine, oracle, n1, m, n2, n3):
    A = oracle.random_tensor(n1, m, n3, 40)
    B = oracle.random_tensor(m, n2, n3, 41)
    M = oracle.random_matrix(n3, n3, 42) + 3.0 * np.eye(n3)   # well conditioned
    got = engine.star_m_product(A, B, M)
    want = oracle.star_m_product(A, B, M)
    assert np.linalg.norm(got - want) <= 1e-11 * np.linalg.norm(want)


def test_hosvd_kats(engine, oracle):
    # tests/test_decompositions.cpp:203-232
    A = oracle.random_tensor(4, 3, 5, 48)
    f = engine.hosvd(A, 4, 3, 5)
    assert np.linalg.norm(A - engine.hosvd_reconstruct(f)) <= 1e-10 * np.linalg.norm(A)
    for U, n in ((f.u1, 4), (f.u2, 3), (f.u3, 5)):
        assert np.linalg.norm(U.T @ U - np.eye(n)) <= 1e-10 * n
    x, y, z = oracle.random_matrix(4, 1, 1), oracle.random_matrix(3, 1, 2), oracle.random_matrix(5, 1, 3)
    R = np.einsum("i,j,k->ijk", x[:, 0], y[:, 0], z[:, 0])
    assert np.linalg.norm(R - engine.hosvd_reconstruct(engine.hosvd(R, 1, 1, 1))) <= 1e-10 * np.linalg.norm(R)
    C = counterexample()
    err = np.linalg.norm(C - engine.hosvd_reconstruct(engine.hosvd(C, 2, 2, 1)))
    assert abs(err * err - 2.0) <= 1e-12
    for bad in ((0, 1, 1), (1, 4, 1)):
        with pytest.raises(engine.ArgumentError):
            engine.hosvd(A, *bad)


@pytest.mark.parametrize("shape,ks", [((12, 9, 14), (5, 4, 6)), ((30, 24, 20), (30, 24, 20)),
                                      ((200, 180, 170), (20, 16, 12)), ((6, 5, 40), (6, 5, 40))])
def test_hosvd_vs_oracle(engine, oracle, shape, ks):
    A = oracle.random_tensor(*shape, 50)
    f = engine.hosvd(A, *ks)
    core, U1, U2, U3 = oracle.hosvd(A, *ks)
    nrm = np.linalg.norm(A)
    rec = engine.hosvd_reconstruct(f)
    assert np.linalg.norm(rec - oracle.hosvd_reconstruct(core, U1, U2, U3)) <= 1e-10 * nrm
    assert abs(np.linalg.norm(f.core) - np.linalg.norm(core)) <= 1e-10 * nrm
    # factors agree column by column where the unfolding's spectrum separates them
    for mode, (Ug, Uo) in enumerate(((f.u1, U1), (f.u2, U2), (f.u3, U3)), start=1):
        s = np.linalg.svd(oracle.mode_unfold(A, mode), compute_uv=False)
        s = np.concatenate([s, np.zeros(Ug.shape[0])])
        for j in range(Ug.shape[1]):
            gap = min(s[j - 1] - s[j] if j else np.inf, s[j] - s[j + 1]) / s[0]
            if gap >= 1e-6 and s[j] > 1e-8 * s[0]:
                assert np.abs(Ug[:, j] - Uo[:, j]).max() <= 1e-8, (mode, j)


def test_matrix_svd_baseline_vs_oracle(engine, oracle):
    # tests/test_decompositions.cpp:234-255
    A = oracle.random_tensor(3, 4, 5, 49)
    assert engine.matrix_svd_baseline(A, 4).error <= 1e-10 * np.linalg.norm(A)
    mb = engine.matrix_svd_baseline(counterexample(), 1)
    assert mb.s.shape == (1,) and abs(mb.s[0] - SQ2) <= 1e-12 and abs(mb.error ** 2 - 2.0) <= 1e-12
    assert engine.matrix_svd_baseline(np.zeros((2, 3, 2)), 2).error == 0.0
    for k in (0, 5):
        with pytest.raises(engine.ArgumentError):
            engine.matrix_svd_baseline(A, k)
    for shape, k in (((20, 30, 8), 6), ((60, 200, 30), 12)):
        A = oracle.random_tensor(*shape, 51)
        got = engine.matrix_svd_baseline(A, k)
        U, s, V, err = oracle.matrix_svd_baseline(A, k)
        nrm = np.linalg.norm(A)
        assert np.abs(got.s - s).max() <= 1e-10 * s[0]
        assert abs(got.error - err) <= 1e-10 * nrm
        assert abs(engine.matrix_svd_error(A, k) - err) <= 1e-10 * nrm
        sf = np.linalg.svd(np.concatenate([A[:, :, z] for z in range(shape[2])]), compute_uv=False)
        for j in range(k):
            gap = min(sf[j - 1] - sf[j] if j else np.inf, sf[j] - sf[j + 1]) / sf[0]
            if gap >= 1e-6:
                assert np.abs(got.u[:, j] - U[:, j]).max() <= 1e-8
                assert np.abs(got.v[:, j] - V[:, j]).max() <= 1e-8


# ------------------------------------------------ Ozaki INT8 Gram (tcgen05 kind::i8)
def _gram_parts(L, T, rows, n3):
    import ctypes as C
    import torch
    c, ch = C.c_int64(), C.c_int64()
    assert L.ppc_gram_plan(rows, n3, C.byref(c), C.byref(ch)) == 0
    parts = torch.empty(c.value * n3 * n3, dtype=torch.float64, device="cuda")
    assert L.ppc_gram_partials(C.c_void_p(T.data_ptr()), rows, rows, n3, ch.value, c.value,
                               C.c_void_p(parts.data_ptr()), 1) == 0, L.ppc_last_error()
    torch.cuda.synchronize()
    return parts.view(c.value, n3, n3).clone(), ch.value


@pytest.mark.parametrize("rows,n3,kind", [(1 << 18, 512, "gauss"), (1 << 22, 512, "cp")])
def test_ozaki_gram_vs_dmma(engine, rows, n3, kind):
    """The INT8 Ozaki Gram (7 digits) against the FP64 DMMA SYRK: agreement to
    ~1e-14 of max|G|, exact symmetry, bitwise determinism, and the plan-chunk
    partials tile the same way on every call (row 8e sharding invariant)."""
    import torch
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    if kind == "gauss":
        T = synth.gaussian_device(rows, 1, n3, 5, 1).reshape(rows, n3)
    else:
        T = synth.cp_tensor_device(1 << 11, rows >> 11, n3, rank=50, noise=1e-3, seed=2).reshape(rows, n3)
    try:
        assert L.ppc_set_ozaki(1) == 0
        L.ppc_timing_enable(1)
        oz, chunk = _gram_parts(L, T, rows, n3)
        import ctypes as C
        buf = C.create_string_buffer(1 << 16)
        L.ppc_timing_report(buf, len(buf), 1)
        L.ppc_timing_enable(0)
        assert "ozaki_syrk" in buf.value.decode(), "Ozaki path not taken"
        oz2, _ = _gram_parts(L, T, rows, n3)
        assert torch.equal(oz, oz2)
        assert L.ppc_set_ozaki(0) == 0
        dm, _ = _gram_parts(L, T, rows, n3)
    finally:
        L.ppc_set_ozaki(1)
    G_oz, G_dm = oz.sum(0), dm.sum(0)
    rel = ((G_oz - G_dm).abs().max() / G_dm.abs().max()).item()
    assert rel <= 1e-13, rel
    for c in range(oz.shape[0]):
        assert torch.equal(oz[c], oz[c].T)
    w_dm = torch.linalg.eigvalsh(G_dm).flip(0)[:16]
    w_oz = torch.linalg.eigvalsh(G_oz).flip(0)[:16]
    assert ((w_dm - w_oz).abs().max() / w_dm[0]).item() <= 1e-13


def test_ozaki_data_q_vs_numpy(engine):
    """data_dependent_transform through the Ozaki Gram (cfg5 distribution,
    512x512 pixels, n3 = 512) against LAPACK on the host: eigenvalue parity
    (SURVEY 8c rule 5) and captured energy."""
    import torch
    a = synth.cp_tensor_device(512, 512, 512, rank=50, noise=1e-3, seed=4)
    t = engine.data_dependent_transform(a, 64)
    T = a.permute(2, 1, 0).reshape(512, -1).T.cpu().numpy()  # tube matrix (N x n3)
    G = T.T @ T
    w = np.linalg.eigvalsh(G)[::-1]
    q = t.q
    lam = np.einsum("ij,ij->j", q, G @ q)
    assert np.abs(lam - w[:64]).max() <= 1e-12 * w[0]
    assert abs(lam.sum() - w[:64].sum()) <= 1e-12 * w[:64].sum()
    assert np.linalg.norm(q.T @ q - np.eye(64)) <= 1e-12


@pytest.mark.parametrize("n1,m,n2,n3,p", [(300, 96, 140, 40, 12), (1024, 512, 1024, 256, 64)])
def test_star_q_host_pipeline_bitwise(engine, n1, m, n2, n3, p):
    """ppc_star_q_product on host buffers (B chunks transformed as they land,
    A row blocks up / C row blocks down on separate copy streams) equals the
    device-resident product bitwise."""
    A = synth.gaussian_device(n1, m, n3, 8, 1)
    B = synth.gaussian_device(m, n2, n3, 8, 2)
    t = engine.Transform("dct", n3, p)
    dev = engine.to_host(engine.star_q_product(A, B, t))
    host = engine.star_q_product(engine.to_host(A), engine.to_host(B), t)
    assert np.array_equal(host, dev)


def test_ozaki_compress_matches_dmma(engine):
    """ppc_tsvdq_compress with the INT8 (Ozaki) Gram, slice Grams and filter
    products against the all-FP64-DMMA run (cfg5 distribution): relative
    error and singular values agree to ~1e-12, the basis on its
    well-separated (signal) columns to ~1e-9."""
    import ctypes as C
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    n1, n2, n3, p, k = 512, 512, 512, 64, 16
    a = synth.cp_tensor_device(n1, n2, n3, rank=50, noise=1e-3, seed=6)
    res = {}
    try:
        for mode in (1, 0):
            assert L.ppc_set_ozaki(mode) == 0
            L.ppc_timing_enable(1)
            Q, U, S, V = (engine.empty_device(sh) for sh in ((n3, p), (n1, k, p), (k, p), (n2, k, p)))
            re = C.c_double()
            rc = L.ppc_tsvdq_compress(C.c_void_p(a.data_ptr()), n1, n2, n3, p, k, C.c_void_p(Q.data_ptr()), None,
                                      C.c_void_p(U.data_ptr()), C.c_void_p(S.data_ptr()), C.c_void_p(V.data_ptr()),
                                      C.byref(re), 1)
            buf = C.create_string_buffer(1 << 16)
            L.ppc_timing_report(buf, len(buf), 1)
            L.ppc_timing_enable(0)
            assert rc == 0, L.ppc_last_error()
            res[mode] = (re.value, engine.to_host(S), engine.to_host(Q), buf.value.decode())
    finally:
        L.ppc_set_ozaki(1)
    assert "ozaki_syrk" in res[1][3], res[1][3]
    assert "ozaki_syrk" not in res[0][3]
    assert abs(res[1][0] - res[0][0]) <= 1e-11 * res[0][0], (res[1][0], res[0][0])
    # signal slices (the noise columns of Q are not determined to the last
    # bits on a plateau, so their slices differ with the basis)
    assert np.abs(res[1][1][:, :40] - res[0][1][:, :40]).max() <= 1e-11 * res[0][1].max()
    assert np.abs(res[1][2][:, :40] - res[0][2][:, :40]).max() <= 1e-9
    # with a shared basis every slice (noise ones too) agrees to 1e-10 per value
    t = engine.Transform.custom(res[0][2])
    s_on = engine.to_host(engine.tsvdq(a, t, k).s)
    try:
        assert L.ppc_set_ozaki(0) == 0
        s_off = engine.to_host(engine.tsvdq(a, t, k).s)
    finally:
        L.ppc_set_ozaki(1)
    assert np.abs(s_on - s_off).max() <= 1e-10 * np.abs(s_off).max()
    assert (np.abs(s_on - s_off) <= 1e-10 * s_off).all()


def test_ozaki_gram_edge_columns(engine):
    """The INT8 Gram with per-column scales across 1e-300 .. 1e+150 magnitudes,
    subnormal and all-zero columns, against the FP64 DMMA SYRK."""
    import torch
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    rows, n3 = 1 << 18, 512
    T = synth.gaussian_device(rows, 1, n3, 9, 1).reshape(rows, n3).clone()
    scales = torch.logspace(-300, 150, n3, dtype=torch.float64, device="cuda")
    T = T * scales
    T[:, 7] = 0.0
    T[:, 11] = 4.9e-324 * torch.sign(T[:, 11])  # subnormal
    T = T.T.contiguous().T  # Fortran layout
    try:
        assert L.ppc_set_ozaki(1) == 0
        oz, _ = _gram_parts(L, T, rows, n3)
        assert L.ppc_set_ozaki(0) == 0
        dm, _ = _gram_parts(L, T, rows, n3)
    finally:
        L.ppc_set_ozaki(1)
    Go, Gd = oz.sum(0), dm.sum(0)
    assert torch.isfinite(Go).all()
    # compare relative to each entry's natural scale sqrt(G_aa G_bb)
    d = torch.sqrt(torch.clamp(torch.diagonal(Gd), min=0))
    denom = torch.outer(d, d) + 1e-300
    rel = ((Go - Gd).abs() / denom)
    mask = denom > 1e-290
    assert rel[mask].max().item() <= 1e-13
    assert (Go[7] == 0).all() and (Go[:, 7] == 0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("shape,val", [((256, 256, 256), float("nan")), ((256, 256, 256), float("inf")),
                                       ((24, 20, 16), float("nan")), ((24, 20, 16), float("-inf"))])
def test_nonfinite_input_rejected(engine, shape, val):
    """The svd guard (matrix_kernels.cpp:32): NaN / Inf anywhere in the input
    fails data_dependent_transform and compress_tsvdq with NumericError —
    through the finiteness flag of the Ozaki Gram's split pass (256^3: the
    INT8 Gram path) and through the plain scan (small shape: DMMA Gram)."""
    n1, n2, n3 = shape
    a = synth.cp_tensor_device(n1, n2, n3, rank=5, noise=1e-3, seed=1)
    a[n1 // 3, n2 - 1, n3 // 2] = val  # one bad value deep inside a late chunk
    with pytest.raises(engine.NumericError):
        engine.data_dependent_transform(a, 8)
    with pytest.raises(engine.NumericError):
        engine.compress_tsvdq(a, 8, 4)
    with pytest.raises(engine.NumericError):  # host input: the slab-streamed Gram
        engine.compress_tsvdq(engine.to_host(a), 8, 4)
    a[n1 // 3, n2 - 1, n3 // 2] = 0.0
    t = engine.data_dependent_transform(a, 8)  # clean input passes again
    assert np.isfinite(t.q).all()


@pytest.mark.gpu
@pytest.mark.parametrize("M,K,N,alpha", [(4096, 64, 256, 0.75), (1000, 40, 96, 1.0), (258, 33, 32, -2.0)])
def test_star_inverse_vs_numpy(engine, M, K, N, alpha):
    """ppc_star_inverse (the star product's inverse transform on the INT8
    tensor cores, row-wise digit split, B resident in shared memory, TMA-store
    epilogue) against numpy FP64: <= 1e-12 relative (Frobenius; the star
    product's tolerance, DESIGN 5: the 6-digit split carries ~sqrt(K) 2^-45 of
    a row's max, ~2e-13 here, against FP64's ~1e-15), partial last
    tile, K < 64 (zero-padded digits), 1-8 sub-tiles; a row block of the
    input gives those rows bit for bit (row-wise digits); rows with a wide
    dynamic range stay accurate relative to their own norm."""
    import ctypes as C
    import torch
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    g = torch.Generator(device="cuda")
    g.manual_seed(M + K + N)
    A = torch.randn(K, M, dtype=torch.float64, device="cuda", generator=g).t()  # M x K, leading dimension M
    A[3] *= 1e6          # a huge row
    A[5] *= 1e-9         # a tiny row
    A[7, 1] = 1e8        # one dominant entry in a row
    Q = (torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g) / K ** 0.5).t()  # N x K, column-major
    Cout = torch.empty(N, M, dtype=torch.float64, device="cuda").t()
    torch.cuda.synchronize()  # the engine runs on its own stream
    L.ppc_timing_report(C.create_string_buffer(1 << 16), 1 << 16, 1)
    L.ppc_timing_enable(1)
    assert L.ppc_star_inverse(C.c_void_p(A.data_ptr()), M, K, C.c_void_p(Q.data_ptr()), N, C.c_double(alpha),
                              C.c_void_p(Cout.data_ptr())) == 0, L.ppc_last_error()
    buf = C.create_string_buffer(1 << 16)
    L.ppc_timing_report(buf, len(buf), 1)
    L.ppc_timing_enable(0)
    assert L.ppc_synchronize() == 0
    assert "ozaki_star_inv" in buf.value.decode()
    want = alpha * (A.cpu().numpy() @ Q.cpu().numpy().T)
    got = Cout.cpu().numpy()
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    # per row, relative to the row's own scale
    rn = np.linalg.norm(A.cpu().numpy(), axis=1) * abs(alpha)
    assert (np.abs(got - want).max(axis=1) <= 1e-12 * rn).all()
    # a row block (as the host pipeline / a shard computes it): the same bits
    r0, nr = 128, min(512, M - 128) & ~1
    Ab = A[r0:r0 + nr].t().contiguous().t()
    Cb = torch.empty(N, nr, dtype=torch.float64, device="cuda").t()
    torch.cuda.synchronize()
    assert L.ppc_star_inverse(C.c_void_p(Ab.data_ptr()), nr, K, C.c_void_p(Q.data_ptr()), N, C.c_double(alpha),
                              C.c_void_p(Cb.data_ptr())) == 0
    assert L.ppc_synchronize() == 0
    assert torch.equal(Cb, Cout[r0:r0 + nr])
    # an output 8 bytes off 16-byte alignment cannot take the TMA store: the
    # call runs on FP64 DMMA instead, same tolerance
    raw = torch.empty(M * N + 1, dtype=torch.float64, device="cuda")
    assert L.ppc_star_inverse(C.c_void_p(A.data_ptr()), M, K, C.c_void_p(Q.data_ptr()), N, C.c_double(alpha),
                              C.c_void_p(raw.data_ptr() + 8)) == 0, L.ppc_last_error()
    assert L.ppc_synchronize() == 0
    got2 = raw[1:].reshape(N, M).t().cpu().numpy()
    assert np.linalg.norm(got2 - want) <= 1e-12 * np.linalg.norm(want)


class _Stages:
    """Records which engine stages ran (ppc_timing_report)."""

    def __enter__(self):
        import ctypes as C
        from paper_2409_19402_b200 import _lib
        self.L = _lib.lib()
        self.L.ppc_timing_report(C.create_string_buffer(1 << 16), 1 << 16, 1)
        self.L.ppc_timing_enable(1)
        return self

    def __exit__(self, *exc):
        import ctypes as C
        import json
        self.L.ppc_synchronize()
        buf = C.create_string_buffer(1 << 16)
        self.L.ppc_timing_report(buf, len(buf), 1)
        self.L.ppc_timing_enable(0)
        self.names = set(json.loads(buf.value.decode()))
        return False


def _assert_nonfinite_match(got, want, rtol=1e-12):
    """Same NaN and infinity positions (and infinity signs); the finite part
    within rtol of the finite part's norm."""
    assert np.array_equal(np.isnan(got), np.isnan(want))
    assert np.array_equal(np.isposinf(got), np.isposinf(want))
    assert np.array_equal(np.isneginf(got), np.isneginf(want))
    f = np.isfinite(want)
    assert np.linalg.norm(got[f] - want[f]) <= rtol * np.linalg.norm(want[f])


@pytest.mark.gpu
def test_star_inverse_nonfinite_rows(engine):
    """ppc_star_inverse with NaN / infinity in some rows: those rows are
    recomputed on FP64 FMAs (the row split marks them), so the output has the
    FP64 product's NaN / infinity pattern; the other rows stay on the INT8
    path at <= 1e-12."""
    import ctypes as C
    import torch
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    M, K, N, alpha = 1000, 64, 128, 0.5
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    A = torch.randn(K, M, dtype=torch.float64, device="cuda", generator=g).t()
    A[3, 5] = float("nan")
    A[70, 0] = float("inf")
    A[71, 9] = -float("inf")
    A[72, 1], A[72, 2] = float("inf"), -float("inf")
    A[999, 63] = float("nan")
    Q = (torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g) / K ** 0.5).t()
    Cout = torch.empty(N, M, dtype=torch.float64, device="cuda").t()
    torch.cuda.synchronize()
    assert L.ppc_star_inverse(C.c_void_p(A.data_ptr()), M, K, C.c_void_p(Q.data_ptr()), N, C.c_double(alpha),
                              C.c_void_p(Cout.data_ptr())) == 0, L.ppc_last_error()
    assert L.ppc_synchronize() == 0
    with np.errstate(invalid="ignore"):
        want = A.cpu().numpy() @ (alpha * Q.cpu().numpy()).T
    _assert_nonfinite_match(Cout.cpu().numpy(), want)
    assert np.isnan(want[3]).all() and np.isnan(want[999]).all() and not np.isfinite(want[70:73]).any()


@pytest.mark.gpu
@pytest.mark.parametrize("b_inf", [False, True])
def test_star_q_nonfinite_matches_fp64(engine, b_inf):
    """star_q_product at a shape whose facewise and inverse take the INT8
    paths, with a NaN in A (and an infinity in B): the dynamic-range gate
    sends the row block holding the NaN (every block, for B's infinity) to
    FP64 DMMA and the inverse recomputes the non-finite rows, so NaN /
    infinity land where the FP64 chain (star_products.cpp:51-59) puts them;
    device and host input agree."""
    rng = np.random.default_rng(21)
    n1, m, n2, n3, p = 384, 256, 128, 64, 32
    a = np.asfortranarray(rng.standard_normal((n1, m, n3)))
    b = np.asfortranarray(rng.standard_normal((m, n2, n3)))
    a[5, 7, 3] = np.nan
    if b_inf:
        b[9, 11, 20] = np.inf
    t = engine.Transform("dct", n3, p)
    q = t.q
    with _Stages() as st:
        got = engine.to_host(engine.star_q_product(engine.to_device(a), engine.to_device(b), t))
    assert "ozaki_star_inv" in st.names, st.names
    assert ("ozaki_gemm" in st.names) == (not b_inf), st.names
    with np.errstate(invalid="ignore"):
        ah = np.einsum("ijt,tq->ijq", a, q)
        bh = np.einsum("ijt,tq->ijq", b, q)
        ch = np.einsum("ijq,jkq->ikq", ah, bh)
        want = np.einsum("ikq,tq->ikt", ch, q) * t.scale
    assert np.isnan(want[5]).all()
    if b_inf:
        assert not np.isfinite(want[:, 11]).any()
    _assert_nonfinite_match(got, want)
    host = engine.star_q_product(a, b, t)
    assert np.array_equal(host, got, equal_nan=True)


@pytest.mark.gpu
def test_compress_re_identity_matches_direct(engine):
    """ppc_tsvdq_compress takes RE from ||A||^2 - sum s_ij^2 (Eckart-Young
    through the polish) when RE^2 >= 2e-2, from the orthogonal split
    ||A - A_k||^2 = (||A||^2 - ||Ahat||^2) + sum_i ||Ahat_i - U_i S_i V_i^T||^2
    (Q orthonormal; one fused residual pass over Ahat) when 2e-3 <= RE^2 <
    2e-2, and measures it against the reconstruction below; all three must
    equal the directly measured relative_error(A, tsvdq_reconstruct(F)), and
    the slice residual pass runs exactly below RE^2 = 2e-2."""
    import ctypes as C
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    cases = [((256, 192, 128), 32, 8, 1e-3, 20),   # RE ~ 0.3: singular values
             ((192, 160, 96), 64, 4, 1e-2, 20),    # noisy, many noise slices: singular values
             ((128, 128, 64), 48, 16, 1e-2, 20),   # RE^2 ~ 5.7e-3: slice residual pass
             ((128, 96, 64), 32, 12, 1e-2, 16),    # RE^2 ~ 8.4e-3: slice residual pass
             ((128, 128, 64), 48, 24, 1e-9, 20)]   # rank 20 < k: RE ~ 1e-9, direct fallback
    buf = C.create_string_buffer(1 << 16)
    for shape, p, k, noise, rank in cases:
        a = synth.cp_tensor(*shape, rank=rank, noise=noise, seed=5)
        da = engine.to_device(a)
        L.ppc_timing_report(buf, len(buf), 1)
        L.ppc_timing_enable(1)
        f, re = engine.compress_tsvdq(da, p, k)
        L.ppc_timing_report(buf, len(buf), 1)
        L.ppc_timing_enable(0)
        red = engine.tsvdq_relative_error(da, f)
        assert abs(re - red) <= 1e-12 * red, (shape, re, red)
        residual_pass = "slice_residual" in buf.value.decode()
        assert residual_pass == (red * red < 2e-2), (shape, red, residual_pass)


@pytest.mark.gpu
def test_ozaki_forward_transform_noise_slices(engine):
    """ppc_tsvdq_compress reuses the data-driven Q Gram's 7-digit split of A
    for Ahat = A x3 Q^T on the INT8 tensor cores (28 digit pairs). With the
    same basis, every slice's singular values -- the noise slices, whose
    Ahat is ~1e-4 of |A||Q|, included -- must agree with the FP64 DMMA
    transform to 1e-10 per value."""
    import ctypes as C
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    n1, n2, n3, p, k = 512, 512, 512, 64, 16
    a = synth.cp_tensor_device(n1, n2, n3, rank=50, noise=1e-3, seed=8)
    Q, U, S, V = (engine.empty_device(sh) for sh in ((n3, p), (n1, k, p), (k, p), (n2, k, p)))
    re = C.c_double()
    L.ppc_timing_enable(1)
    rc = L.ppc_tsvdq_compress(C.c_void_p(a.data_ptr()), n1, n2, n3, p, k, C.c_void_p(Q.data_ptr()), None,
                              C.c_void_p(U.data_ptr()), C.c_void_p(S.data_ptr()), C.c_void_p(V.data_ptr()),
                              C.byref(re), 1)
    buf = C.create_string_buffer(1 << 16)
    L.ppc_timing_report(buf, len(buf), 1)
    L.ppc_timing_enable(0)
    assert rc == 0, L.ppc_last_error()
    assert "ozaki_fwd" in buf.value.decode(), buf.value.decode()
    s_fwd = engine.to_host(S)
    t = engine.Transform.custom(engine.to_host(Q))
    s_dmma = engine.to_host(engine.tsvdq(a, t, k).s)  # same Q, FP64 DMMA transform
    assert (np.abs(s_fwd - s_dmma) <= 1e-10 * s_dmma).all(), np.max(np.abs(s_fwd - s_dmma) / s_dmma)
    try:
        assert L.ppc_set_ozaki(0) == 0
        s_off = engine.to_host(engine.tsvdq(a, t, k).s)  # everything FP64 DMMA
    finally:
        L.ppc_set_ozaki(1)
    assert (np.abs(s_fwd - s_off) <= 1e-10 * s_off).all(), np.max(np.abs(s_fwd - s_off) / s_off)


def _eig_case(kind, n, seed=0):
    rng = np.random.default_rng(seed)
    if kind == "spiked":  # rank-50 spikes over a Marchenko-Pastur plateau (the cfg5 Gram)
        F = rng.standard_normal((n, 50)) * np.sqrt(np.logspace(9.8, 6, 50))
        Nn = rng.standard_normal((n, 4 * n))
        G = F @ F.T + 4.2 / (4 * n) * (Nn @ Nn.T)
    elif kind == "lowrank":  # zero-eigenvalue cluster inside the wanted set
        F = rng.standard_normal((n, 30))
        G = F @ F.T
    else:  # exactly repeated eigenvalues
        Qr, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = np.concatenate([np.full(40, 5.0), np.full(40, 3.0), np.linspace(1, 0, n - 80)])
        G = (Qr * lam) @ Qr.T
    return 0.5 * (G + G.T)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n,p", [("spiked", 1024, 128), ("lowrank", 512, 48), ("repeated", 300, 100),
                                      ("spiked", 200, 20)])
def test_direct_eigensolver(engine, kind, n, p):
    """ppc_sym_eig_top on one Gram (Householder tridiagonalization, bisection,
    inverse iteration, CholQR3, compact-WY back-transform): eigenvalues within
    1e-13 lambda_1 of LAPACK, orthonormal to 1e-13, residuals 1e-13 lambda_1,
    captured energy to 1e-13, the sign rule, and bitwise repeatable."""
    import ctypes as C
    import torch
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    G = _eig_case(kind, n)
    w = np.linalg.eigvalsh(G)[::-1]
    g = torch.tensor(np.asfortranarray(G).ravel(order="F"), device="cuda")
    outs = []
    for _ in range(2):
        Qd = torch.empty((p, n), dtype=torch.float64, device="cuda")
        Sd = torch.empty(p, dtype=torch.float64, device="cuda")
        assert L.ppc_sym_eig_top(C.c_void_p(g.data_ptr()), n, p, C.c_void_p(Qd.data_ptr()),
                                 C.c_void_p(Sd.data_ptr()), 1) == 0, L.ppc_last_error()
        torch.cuda.synchronize()  # device pointers: the call is stream-ordered on the engine's stream
        outs.append((Qd.cpu().numpy().T.copy(), Sd.cpu().numpy() ** 2))
    (Q, lam), (Q2, lam2) = outs
    assert np.array_equal(Q, Q2) and np.array_equal(lam, lam2)
    l1 = w[0]
    assert np.max(np.abs(lam - w[:p])) <= 1e-13 * l1
    assert np.max(np.abs(Q.T @ Q - np.eye(p))) <= 1e-13
    # residuals: ~1e-15 lambda_1 on separated spectra; the exactly repeated
    # clusters leave ~1e-12 (vectors arbitrary within the eigenspace)
    assert np.max(np.linalg.norm(G @ Q - Q * lam, axis=0)) <= (1e-11 if kind == "repeated" else 1e-13) * l1
    assert abs(np.trace(Q.T @ G @ Q) - w[:p].sum()) <= 1e-13 * w[:p].sum()
    big = np.argmax(np.abs(Q), axis=0)  # matrix_kernels.cpp:16-25
    assert (Q[big, np.arange(p)] >= 0).all()


@pytest.mark.gpu
def test_ozaki_filter_large_slices(engine):
    """Slices of r >= 1024 run the Chebyshev filter and Rayleigh-Ritz G X on
    the INT8 tensor cores (3/4/6 digit levels, upper-triangle streaming of the
    slice Grams): with a shared basis every singular value, noise slices
    included, matches the all-FP64 path to 1e-10 per value."""
    import ctypes as C
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    n1, n2, n3, p, k = 1024, 1024, 256, 16, 8
    a = synth.cp_tensor_device(n1, n2, n3, rank=12, noise=1e-3, seed=12)
    t = engine.data_dependent_transform(a, p)
    L.ppc_timing_enable(1)
    s_on = engine.to_host(engine.tsvdq(a, t, k).s)
    buf = C.create_string_buffer(1 << 16)
    L.ppc_timing_report(buf, len(buf), 1)
    L.ppc_timing_enable(0)
    assert "ozaki_gemm" in buf.value.decode(), buf.value.decode()
    try:
        assert L.ppc_set_ozaki(0) == 0
        s_off = engine.to_host(engine.tsvdq(a, t, k).s)
    finally:
        L.ppc_set_ozaki(1)
    assert (np.abs(s_on - s_off) <= 1e-10 * s_off).all(), np.max(np.abs(s_on - s_off) / s_off)


@pytest.mark.gpu
def test_dist_single_rank_kept_digits_matches_fused(engine):
    """dist.py's per-rank path at a size where the Gram runs on the INT8 path
    over whole 4096-row blocks: the engine keeps the 7-digit split
    (ppc_gram_partials_keep) and the shard's forward transform reuses it
    (ppc_mode3_forward_digits), as the fused ppc_tsvdq_compress does."""
    import torch
    from paper_2409_19402_b200 import dist as pdist
    n1, n2, n3, p, k = 512, 512, 512, 64, 8
    a = synth.cp_tensor_device(n1, n2, n3, rank=30, noise=1e-3, seed=13)
    f, re = engine.compress_tsvdq(a, p, k)
    import ctypes as C
    from paper_2409_19402_b200 import _lib
    L = _lib.lib()
    be = pdist.DeviceBackend("cuda:0")
    plan = pdist.make_plan(n1, n2, n3, p, 1, 0, be)
    L.ppc_timing_enable(1)
    Q, U, S, V, re2 = pdist.sharded_compress(a, plan, k, be)
    torch.cuda.synchronize()
    buf = C.create_string_buffer(1 << 16)
    L.ppc_timing_report(buf, len(buf), 1)
    L.ppc_timing_enable(0)
    assert "ozaki_fwd" in buf.value.decode(), buf.value.decode()  # the kept digits were used
    assert be._kept == 0  # and released
    assert np.array_equal(engine.to_host(Q), f.transform.q)  # same digits, same Gram tree
    np.testing.assert_allclose(engine.to_host(S), engine.to_host(f.s), rtol=1e-12)
    assert abs(re2 - re) <= 1e-12 * re


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_gram_int8_decision_bitwise(engine, world):
    """the INT8-vs-DMMA choice of the Gram is the plan's, not the
    call's. 128 x 256 x 128 has 8 chunks of 4096 rows; at 2 and 4 ranks each
    shard holds 16384 / 8192 rows. Every shard's partials run on the INT8
    path (as the whole-tensor call), and the rank roots finished by the
    pairwise tree give Q bitwise equal to the 1-GPU data-driven basis
    (emulated ranks, one after another, on one GPU)."""
    import ctypes as C
    import torch
    from paper_2409_19402_b200 import _lib, dist as pdist
    n1, n2, n3, p = 128, 256, 128, 16
    a = synth.cp_tensor_device(n1, n2, n3, rank=10, noise=1e-3, seed=21)
    # the compress chain keeps the Gram's 7-digit split for the forward
    # transform, as the shards' ppc_gram_partials_keep does
    want = engine.compress_tsvdq(a, p, 4)[0].transform.q
    be = pdist.DeviceBackend("cuda:0")
    roots = []
    L = _lib.lib()
    for r in range(world):
        plan = pdist.make_plan(n1, n2, n3, p, world, r, be)
        blk = a[:, plan.j0:plan.j0 + plan.nj, :].permute(2, 1, 0).contiguous().permute(2, 1, 0)
        buf = C.create_string_buffer(1 << 16)
        L.ppc_timing_report(buf, len(buf), 1)
        L.ppc_timing_enable(1)
        parts, bad = be.gram_partials(blk, n1 * plan.nj, n3, plan.chunk, plan.chunks_per_rank)
        torch.cuda.synchronize()
        L.ppc_timing_report(buf, len(buf), 1)
        L.ppc_timing_enable(0)
        assert "gram_ozaki" in buf.value.decode(), (r, buf.value.decode())
        assert not bad
        be.release_kept()
        roots.append(be.tree_reduce(parts))
    Q, _ = be.sym_eig_top(pdist._tree_finish(roots), n3, p)
    torch.cuda.synchronize()
    assert np.array_equal(engine.to_host(Q), engine.to_host(want))


@pytest.mark.gpu
def test_sharded_gram_nonfinite_flag(engine):
    """ppc_gram_partials_keep reports a shard's NaN / Inf (the caller combines
    the flags over the ranks, matrix_kernels.cpp:32) on both the INT8 and the
    DMMA Gram paths."""
    import torch
    from paper_2409_19402_b200 import dist as pdist
    be = pdist.DeviceBackend("cuda:0")
    for n3 in (128, 64):  # INT8 / DMMA partials
        a = synth.cp_tensor_device(64, 256, n3, rank=5, noise=1e-3, seed=2)
        chunks, chunk = be.gram_plan(64 * 256, n3)
        _, bad = be.gram_partials(a, 64 * 256, n3, chunk, chunks)
        be.release_kept()
        assert not bad
        a[5, 100, n3 - 1] = float("inf")
        _, bad = be.gram_partials(a, 64 * 256, n3, chunk, chunks)
        be.release_kept()
        torch.cuda.synchronize()
        assert bad, n3


# ------------------------------------- block one-sided Jacobi (large k, K6b)
def _graded(m, n, rng, lo):
    r = min(m, n)
    qu, _ = np.linalg.qr(rng.standard_normal((m, r)))
    qv, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return (qu * np.geomspace(1.0, lo, r)) @ qv.T


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k", [(300, 260, 260), (260, 300, 200), (520, 500, 400)])
def test_block_jacobi_vs_lapack(engine, m, n, k):
    """Slices too large for the one-CTA Jacobi that keep k > r/2 triplets go to
    the blocked one-sided Jacobi (block_jacobi.cu): singular values as LAPACK
    (relative 1e-10 down to 1e-6 sigma_1, also on a graded spectrum), U and V
    orthonormal, the rank-k reconstruction, the sign rule, and a zero and a
    rank-deficient slice (orthonormal completion for zero values)."""
    import ctypes as C
    from paper_2409_19402_b200 import _lib
    rng = np.random.default_rng(m + n + k)
    batch = 4
    a = np.zeros((m, n, batch))
    a[:, :, 0] = rng.standard_normal((m, n))
    a[:, :, 1] = _graded(m, n, rng, 1e-8)
    a[:, :, 2] = rng.standard_normal((m, 7)) @ rng.standard_normal((7, n))  # rank 7 < k
    a = np.asfortranarray(a)  # slice 3: zero
    L = _lib.lib()
    buf = C.create_string_buffer(1 << 16)
    L.ppc_timing_report(buf, len(buf), 1)
    L.ppc_timing_enable(1)
    U, s, V = engine.truncated_svd(a, k)
    L.ppc_timing_report(buf, len(buf), 1)
    L.ppc_timing_enable(0)
    assert "block_jacobi" in buf.value.decode(), buf.value.decode()
    for z in range(batch):
        u_, sn, vt_ = np.linalg.svd(a[:, :, z], full_matrices=False)
        big = sn[:k] >= 1e-6 * max(sn[0], 1e-300)
        np.testing.assert_allclose(s[big, z], sn[:k][big], rtol=1e-10)
        assert np.all(np.abs(s[:, z] - sn[:k]) <= 1e-13 * max(1.0, sn[0])), z
        assert np.linalg.norm(U[:, :, z].T @ U[:, :, z] - np.eye(k)) <= 1e-10 * k, z
        assert np.linalg.norm(V[:, :, z].T @ V[:, :, z] - np.eye(k)) <= 1e-10 * k, z
        rec = (U[:, :, z] * s[:, z]) @ V[:, :, z].T
        want = (u_[:, :k] * sn[:k]) @ vt_[:k]
        assert np.linalg.norm(rec - want) <= 1e-10 * max(1.0, np.linalg.norm(a[:, :, z])), z
        for j in range(k):
            i = int(np.argmax(np.abs(U[:, j, z])))
            assert U[i, j, z] >= 0, (z, j)


def _tsvdq2_select(s_all, gamma):
    """decompositions.cpp:137-167 restated: values above 1e-12 of the global
    max, sorted descending (ties: slice, then position), the shortest prefix
    whose energy reaches gamma of the total."""
    r, p = s_all.shape
    cutoff = 1e-12 * s_all[0].max()
    pool = sorted(((-s_all[j, i], i, j) for i in range(p) for j in range(r) if s_all[j, i] > cutoff))
    e = np.cumsum([v * v for v, _, _ in pool])
    K = min(int(np.searchsorted(e, gamma * e[-1], side="left")) + 1, len(pool))
    mr = np.zeros(p, dtype=np.int64)
    for _, i, _ in pool[:K]:
        mr[i] += 1
    return mr


@pytest.mark.gpu
def test_tsvdq2_large_slices_vs_lapack(engine):
    """tsvdq2 (k = r for every slice) on 1024^2 slices finishes in seconds on
    the blocked Jacobi and matches LAPACK: full spectra, the multirank
    selection, and the reconstruction of the kept triplets."""
    import time
    rng = np.random.default_rng(77)
    n1 = n2 = 1024
    n3, p, gamma = 6, 4, 0.9
    a = np.asfortranarray(rng.standard_normal((n1, n2, n3)) +
                          np.einsum("ir,jr,kr->ijk", rng.standard_normal((n1, 20)), rng.standard_normal((n2, 20)),
                                    rng.standard_normal((n3, 20))))
    t = engine.Transform("dct", n3, p)
    t0 = time.time()
    f = engine.tsvdq2(engine.to_device(a), t, gamma)
    s_all = engine.to_host(f.s)
    assert time.time() - t0 < 60
    ah = np.einsum("ijk,kl->ijl", a, t.q)
    sn = np.stack([np.linalg.svd(ah[:, :, i], compute_uv=False) for i in range(p)], axis=1)
    mr = np.asarray(f.multirank)
    assert np.array_equal(mr, _tsvdq2_select(sn, gamma))
    for i in range(p):  # kept values (the factors are zero beyond multirank[i])
        np.testing.assert_allclose(s_all[:mr[i], i], sn[:mr[i], i], rtol=1e-10)
        assert not s_all[mr[i]:, i].any()
    u, v = engine.to_host(f.u), engine.to_host(f.v)
    for i in range(p):
        kk = int(f.multirank[i])
        uu, ss, vt = np.linalg.svd(ah[:, :, i], full_matrices=False)
        rec = (u[:, :kk, i] * s_all[:kk, i]) @ v[:, :kk, i].T
        assert np.linalg.norm(rec - (uu[:, :kk] * ss[:kk]) @ vt[:kk]) <= 1e-10 * np.linalg.norm(ah[:, :, i])


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,world", [(1024, 128, 8), (512, 32, 4), (300, 20, 2)])
def test_sharded_eigensolve_bitwise(engine, n, p, world):
    """The data-driven Q's eigensolve split across ranks (dist.sharded_eig:
    tridiagonalization replicated, eigenvalues / inverse iteration and the
    back-transformation sharded by index, ppc_sym_eig_split_*) gives Q bitwise
    equal to the 1-GPU solve (ppc_sym_eig_top). Emulated ranks, one after
    another, on one GPU."""
    import torch
    from paper_2409_19402_b200 import dist as pdist
    g = torch.Generator(device="cuda")
    g.manual_seed(n + p)
    Y = torch.randn(4 * n, n, dtype=torch.float64, device="cuda", generator=g)
    Y[:, :40] *= torch.linspace(30.0, 3.0, 40, dtype=torch.float64, device="cuda")  # spikes over a plateau
    Gm = (Y.t() @ Y).contiguous()
    be = pdist.DeviceBackend("cuda:0")
    want, _ = be.sym_eig_top(Gm, n, p)
    h = be.eig_begin(Gm, n, p)
    assert h is not None
    try:
        ps = p // world
        Zall = torch.cat([be.eig_vectors(h, n, r * ps, (r + 1) * ps) for r in range(world)], dim=1)
        Zall = Zall.permute(1, 0).contiguous().permute(1, 0)
        Q = torch.cat([be.eig_finish(h, Zall.clone(), n, r * ps, (r + 1) * ps) for r in range(world)], dim=1)
    finally:
        be.eig_release(h)
    torch.cuda.synchronize()
    assert torch.equal(Q, want)
    # and it is the eigenbasis: captured energies vs LAPACK's eigenvalues
    lam = np.sort(np.linalg.eigvalsh(Gm.cpu().numpy()))[::-1][:p]
    cap = torch.sum(Q * (Gm @ Q), dim=0).cpu().numpy()
    assert np.max(np.abs(cap - lam)) <= 1e-12 * lam[0]


def test_concurrent_host_threads_match_serial(engine, oracle):
    """The engine keeps its device context, streams, workspace cache and stage
    timers per host thread (the reference's slice loops run on worker threads,
    parallel.cpp:29-57): four threads calling the C-ABI at once get the bits of
    the same calls made one after another."""
    import threading
    pp = engine
    t = pp.Transform("dct", 48, 12)
    inputs = [oracle.random_tensor(96, 80, 48, 100 + i) for i in range(4)]

    def work(a):
        at = np.asfortranarray(a.transpose(1, 0, 2))
        c = pp.star_q(a, at, t)
        f = pp.tsvdq(a, t, 5)
        fq, re = pp.compress_tsvdq(a, 12, 5)
        return c, f.s, re, fq.transform.q

    serial = [work(a) for a in inputs]
    out = [None] * 4
    errs = []

    def run(i):
        try:
            for _ in range(3):
                out[i] = work(inputs[i])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for got, want in zip(out, serial):
        assert np.array_equal(got[0], want[0])
        assert np.array_equal(got[1], want[1])
        assert got[2] == want[2]
        assert np.array_equal(got[3], want[3])


def test_star_q_algebra_and_error_identities_random_instances(engine, oracle):
    """Property checks in the spirit of the reference's verify suite
    (src/verify.cpp:487-537, 581-726: star-Q algebra, projection tail,
    Eckart-Young identity, recovery), on the GPU path over random instances
    and all four transform kinds."""
    pp = engine
    rng = np.random.default_rng(11)
    worst = 0.0
    for inst in range(16):
        n1, m, n2, l = (int(rng.integers(2, 9)) for _ in range(4))
        n3 = int(rng.choice([4, 6, 8, 12]))
        p = int(rng.integers(1, n3 + 1))
        kind = ["dct", "haar", "random", "data"][inst % 4]
        A = np.asfortranarray(rng.standard_normal((n1, m, n3)))
        B = np.asfortranarray(rng.standard_normal((m, n2, n3)))
        B2 = np.asfortranarray(rng.standard_normal((m, n2, n3)))
        Cc = np.asfortranarray(rng.standard_normal((n2, l, n3)))
        if kind == "haar":  # the reference's Haar basis exists for n3 = 2 and 4 only (transforms.cpp:45-60)
            n3 = 4
            p = min(p, n3)
            A, B, B2, Cc = (np.asfortranarray(x[:, :, :4]) for x in (A, B, B2, Cc))
        t = pp.data_dependent_transform(A, p) if kind == "data" else pp.Transform(kind, n3, p, seed=inst)
        q = t.q
        nrm = lambda x: float(np.linalg.norm(x))  # noqa: E731
        AB = pp.star_q(A, B, t)
        # associativity, distributivity
        lhs, rhs = pp.star_q(AB, Cc, t), pp.star_q(A, pp.star_q(B, Cc, t), t)
        worst = max(worst, nrm(lhs - rhs) / max(nrm(lhs), 1e-300))
        worst = max(worst, nrm(pp.star_q(A, np.asfortranarray(B + B2), t) - AB - pp.star_q(A, B2, t)) / nrm(AB))
        # transpose reversal, identity from both sides (the identity acts as the projection)
        tr = pp.star_q_transpose(AB, t)
        worst = max(worst, nrm(tr - pp.star_q(pp.star_q_transpose(B, t), pp.star_q_transpose(A, t), t)) / nrm(tr))
        PA = oracle.mode3_product(A, q @ q.T)
        worst = max(worst, nrm(pp.star_q(pp.star_q_identity(n1, t), A, t) - PA) / nrm(A))
        worst = max(worst, nrm(pp.star_q(A, pp.star_q_identity(m, t), t) - PA) / nrm(A))
        # projection form: the product only sees the projected parts of its factors
        PB = oracle.mode3_product(B, q @ q.T)
        worst = max(worst, nrm(pp.star_q(PA, PB, t) - AB) / nrm(AB))
        # transform-domain slices of the product are the facewise products
        worst = max(worst, nrm(oracle.mode3_product(AB, q.T) -
                               pp.facewise_product(oracle.mode3_product(A, q.T), oracle.mode3_product(B, q.T))) /
                    nrm(AB))
        # Eckart-Young identity and projection tail for every k
        T = A.reshape(-1, n3, order="F")
        sv = np.linalg.svd(T, compute_uv=False)
        for k in range(1, min(n1, m) + 1):
            f = pp.tsvdq(A, t, k)
            tot, ey, pr = pp.tsvdq_error(A, f)
            worst = max(worst, abs(tot ** 2 - ey ** 2 - pr ** 2) / nrm(A) ** 2)
            if kind == "data":
                tail = float(np.sum(sv[p:] ** 2))
                worst = max(worst, abs(pr ** 2 - tail) / nrm(A) ** 2)
            # the kept slice spectra are the leading singular values of the transform-domain slices
            ah = oracle.mode3_product(A, q.T)
            for i in range(p):
                si = np.linalg.svd(ah[:, :, i], compute_uv=False)[:k]
                worst = max(worst, float(np.max(np.abs(f.s[:, i] - si))) / max(si[0], 1e-300))
        # recovery: rank-r slices in the transform domain come back exactly at k = r
        r = 1 + inst % 2
        core = np.zeros((n1, m, p), order="F")
        for i in range(p):
            core[:, :, i] = rng.standard_normal((n1, r)) @ rng.standard_normal((r, m))
        X = oracle.mode3_product(core, q)
        fx = pp.tsvdq(X, t, min(r, n1, m))
        worst = max(worst, pp.tsvdq_relative_error(X, fx) if min(n1, m) >= r else 0.0)
    assert worst <= 1e-10, worst


def test_projection_and_truncation_optimality(engine, oracle):
    """verify.cpp:513-537 and the Eckart-Young optimality check: the
    data-driven Q's projection error is no larger than that of random Stiefel
    samples of the same p, and tsvdq's rank-k truncation error no larger than
    that of random facewise rank-k approximations in the transform domain."""
    pp = engine
    rng = np.random.default_rng(23)
    for inst in range(4):
        n1, n2, n3 = int(rng.integers(4, 10)), int(rng.integers(4, 10)), int(rng.integers(4, 10))
        p, k = int(rng.integers(1, n3)), int(rng.integers(1, min(n1, n2)))
        A = np.asfortranarray(rng.standard_normal((n1, n2, n3)))
        t = pp.data_dependent_transform(A, p)
        best = pp.projection_error(A, t)
        for s in range(20):
            tr = pp.Transform("random", n3, p, seed=1000 * inst + s)
            assert best <= pp.projection_error(A, tr) * (1 + 1e-12)
        f = pp.tsvdq(A, t, k)
        _, ey, _ = pp.tsvdq_error(A, f)
        ah = oracle.mode3_product(A, t.q.T)
        for s in range(20):
            err2 = 0.0
            for i in range(p):
                R = rng.standard_normal((k, n2))  # a random k-dimensional row space
                # the best fit within it: least squares on the left factor
                coef, *_ = np.linalg.lstsq(R.T, ah[:, :, i].T, rcond=None)
                err2 += np.linalg.norm(ah[:, :, i] - coef.T @ R) ** 2
            assert ey ** 2 <= err2 * (1 + 1e-12)
