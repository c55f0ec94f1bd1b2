"""Pin the CPU oracle (oracle/ppo.c) against every known-answer test the
reference holds for the hot path and against an
independent LAPACK (numpy) computation. CPU only."""
import math

import numpy as np
import pytest

from oracle import ppo

SQ2 = math.sqrt(2.0)


def tube(v):
    return np.asarray(v, dtype=float).reshape(1, 1, -1)


def counterexample():
    # tests/support/common.hpp:15-22
    a = np.zeros((2, 2, 2))
    a[:, :, 0] = np.eye(2)
    a[:, :, 1] = np.diag([1.0, -1.0])
    return a


def test_star_q_worked_tube():
    # tests/test_star_products.cpp:70-78; verify.cpp:133-157
    a, b = tube([2, 4, 6, 8]), tube([1, -1, 1, 0])
    np.testing.assert_allclose(ppo.star_q_product(a, b, ppo.haar_q(4, 2)).ravel(), [3, 3, 3, 0],
                               atol=1e-12)
    h4 = ppo.haar_q(4, 4)
    np.testing.assert_allclose(ppo.star_q_product(a, b, h4[:, 2:]).ravel(), [-1, 1, 0, 8],
                               atol=1e-12)


def test_mode3_haar_projection():
    # tests/test_tensor.cpp:101-121
    a = tube([2, 4, 6, 8])
    q = ppo.haar_q(4, 2)
    ahat = ppo.mode3_product(a, q.T).ravel()
    assert ahat[0] == pytest.approx(3 + 3 * SQ2, rel=1e-14)
    assert ahat[1] == pytest.approx(3 - 3 * SQ2, rel=1e-14)
    np.testing.assert_allclose(ppo.mode3_product(a, q @ q.T).ravel(), [3, 3, 6, 0], atol=1e-12)
    b = tube([1, -1, 1, 0])
    np.testing.assert_allclose(ppo.mode3_product(b, q @ q.T).ravel(), [0, 0, 1, 0], atol=1e-12)


def test_projection_error_kat():
    # tests/test_transforms.cpp:112-121
    assert ppo.projection_error(tube([2, 4, 6, 8]), ppo.haar_q(4, 2)) == pytest.approx(
        math.sqrt(66.0), abs=1e-12)
    g = ppo.random_tensor(3, 4, 4, 21)
    assert ppo.projection_error(g, ppo.haar_q(4, 4)) <= 1e-10


def test_error_split_counterexample():
    # tests/test_decompositions.cpp:61-78; verify.cpp:177-191
    a = counterexample()
    q, _, _ = ppo.data_dependent_q(a, 1)
    U, S, V = ppo.tsvdq(a, q, 1)
    t, e, p = ppo.tsvdq_error(a, U, S, V, q)
    assert abs(t - math.sqrt(3.0)) <= 1e-12
    assert abs(e - 1.0) <= 1e-12
    assert abs(p - SQ2) <= 1e-12
    qh = ppo.haar_q(2, 1)
    U, S, V = ppo.tsvdq(a, qh, 1)
    t, e, p = ppo.tsvdq_error(a, U, S, V, qh)
    assert abs(t - SQ2) <= 1e-12 and abs(e) <= 1e-12 and abs(p - SQ2) <= 1e-12
    # Ahat_0 = [[sqrt2, 0], [0, 0]]
    ah = ppo.mode3_product(a, qh.T)[:, :, 0]
    np.testing.assert_allclose(ah, [[SQ2, 0], [0, 0]], atol=1e-12)
    # tests/test_metrics.cpp:19-24
    rec = ppo.tsvdq_reconstruct(U, S, V, qh)
    assert abs(ppo.relative_error(a, rec) - SQ2 / 2) <= 1e-12


def test_facewise_tube_product():
    # tests/test_tensor.cpp:144-149
    ab = ppo.facewise_product(tube([1, 2, 3]), tube([4, 5, -6])).ravel()
    assert list(ab) == [4.0, 10.0, -18.0]


def test_dct_constant_tube():
    # tests/test_transforms.cpp:51-56
    q = ppo.dct_q(4, 4)
    hat = q.T @ np.full(4, -2.5)
    assert abs(hat[0] - (-2.5 * 2.0)) <= 1e-12
    assert np.all(np.abs(hat[1:]) <= 1e-12)
    one = ppo.dct_q(6, 1)
    assert np.all(np.abs(one[:, 0] - 1 / math.sqrt(6)) <= 1e-14)


def test_data_q_rank_one_mode3():
    # tests/test_transforms.cpp:70-81
    v = np.array([1 / 3, 2 / 3, 2 / 3])
    c = ppo.random_matrix(2, 2, 5)
    b = c[:, :, None] * v[None, None, :]
    q, _, _ = ppo.data_dependent_q(b, 1)
    assert min(np.linalg.norm(q[:, 0] - v), np.linalg.norm(q[:, 0] + v)) <= 1e-12
    q2, _, _ = ppo.data_dependent_q(counterexample(), 2)
    aq = np.abs(q2)
    assert np.abs(aq - np.eye(2)).max() <= 1e-12 or np.abs(aq - np.eye(2)[::-1]).max() <= 1e-12
    g = ppo.random_tensor(4, 3, 5, 11)
    qf, _, _ = ppo.data_dependent_q(g, 5)
    assert ppo.projection_error(g, qf) <= 1e-10


def test_full_k_full_p_lossless_and_projection():
    # tests/test_decompositions.cpp:80-103
    rng_a = ppo.random_tensor(4, 3, 5, 42)
    full = ppo.random_orthogonal_q(5, 5, 9)
    U, S, V = ppo.tsvdq(rng_a, full, 3)
    nrm = np.linalg.norm(rng_a)
    assert np.linalg.norm(rng_a - ppo.tsvdq_reconstruct(U, S, V, full)) <= 1e-10 * nrm
    t, e, p = ppo.tsvdq_error(rng_a, U, S, V, full)
    assert t <= 1e-10 * nrm and e <= 1e-10 * nrm and p <= 1e-10 * nrm
    part = ppo.random_orthogonal_q(5, 3, 9)
    U, S, V = ppo.tsvdq(rng_a, part, 3)
    proj = ppo.mode3_product(rng_a, part @ part.T)
    assert np.linalg.norm(proj - ppo.tsvdq_reconstruct(U, S, V, part)) <= 1e-10 * nrm


def test_exact_rank_only_projection_error():
    # tests/test_decompositions.cpp:105-116 (exact-rank construction)
    q = ppo.random_orthogonal_q(6, 4, 17)
    hat = np.zeros((5, 4, 4), order="F")
    for s in range(4):
        x = ppo.random_matrix(5, 2, 100 + s)
        y = ppo.random_matrix(4, 2, 200 + s)
        hat[:, :, s] = x @ y.T
    a = ppo.mode3_product(hat, q)
    U, S, V = ppo.tsvdq(a, q, 2)
    t, e, p = ppo.tsvdq_error(a, U, S, V, q)
    nrm = np.linalg.norm(a)
    assert abs(t - p) <= 1e-10 * nrm and e <= 1e-10 * nrm and t <= 1e-10 * nrm


def test_p_equals_n3_star_m_and_scale_law():
    # tests/test_star_products.cpp:80-102
    a = ppo.random_tensor(3, 2, 5, 70)
    b = ppo.random_tensor(2, 4, 5, 71)
    q = ppo.random_orthogonal_q(5, 5, 42)
    got = ppo.star_q_product(a, b, q)
    # star_m with M = Q^T: ((A x3 M) facewise (B x3 M)) x3 M^{-1}, M^{-1} = Q
    ah = np.einsum("ijk,lk->ijl", a, q.T)
    bh = np.einsum("ijk,lk->ijl", b, q.T)
    ch = np.einsum("imk,mjk->ijk", ah, bh)
    want = np.einsum("ijk,lk->ijl", ch, q)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    qd = ppo.dct_q(4, 2)
    a2, b2 = ppo.random_tensor(2, 2, 4, 80), ppo.random_tensor(2, 3, 4, 81)
    base = ppo.star_q_product(a2, b2, qd)
    for c in (-2.0, 0.5, 3.0):
        assert np.linalg.norm(ppo.star_q_product(a2, b2, qd, c) - c * base) <= 1e-12 * abs(c) * np.linalg.norm(base)


def test_ey_identity_and_projection_tail():
    # verify.cpp:702-726 (EY identity) and :487-511 (projection tail, Q = U3)
    a = ppo.random_tensor(6, 5, 7, 7)
    q = ppo.dct_q(7, 4)
    U, S, V = ppo.tsvdq(a, q, 3)
    t, e, p = ppo.tsvdq_error(a, U, S, V, q)
    assert abs(t * t - (e * e + p * p)) <= 1e-10 * np.sum(a * a)
    qd, sig, _ = ppo.data_dependent_q(a, 4)
    unf = a.reshape(30, 7, order="F").T
    s_all = np.linalg.svd(unf, compute_uv=False)
    tail = np.sum(s_all[4:] ** 2)
    assert abs(ppo.projection_error(a, qd) ** 2 - tail) <= 1e-9 * tail


def test_svd_contract_and_pins():
    # verify.cpp:317-362; tests/test_matrix_kernels.cpp:11-47
    a = ppo.random_matrix(7, 5, 21)
    U, s, V = ppo.svd(a)
    assert np.all(np.diff(s) <= 0) and s[-1] >= 0
    assert np.linalg.norm(U.T @ U - np.eye(5)) <= 5e-10
    assert np.linalg.norm(V.T @ V - np.eye(5)) <= 5e-10
    assert np.linalg.norm(a - U @ np.diag(s) @ V.T) <= 1e-10 * np.linalg.norm(a)
    for j in range(5):  # sign rule
        i = int(np.argmax(np.abs(U[:, j])))
        assert U[i, j] >= 0
    U, s, V = ppo.svd(np.array([[SQ2, 0], [0, 0]]))
    assert s[0] == pytest.approx(SQ2, rel=1e-14) and abs(s[1]) <= 1e-14
    _, s, _ = ppo.svd(np.eye(3))
    np.testing.assert_allclose(s, 1.0, rtol=1e-14)
    sn = np.linalg.svd(a, compute_uv=False)
    _, s, _ = ppo.svd(a)
    np.testing.assert_allclose(s, sn, rtol=1e-13)


def test_errors_mirror_reference():
    with pytest.raises(ppo.OracleError) as e:
        ppo.tsvdq(np.ones((2, 2, 2)), ppo.haar_q(2, 1), 7)
    assert e.value.kind == "argument_error"
    with pytest.raises(ppo.OracleError) as e:
        ppo.relative_error(np.zeros((2, 2, 2)), np.zeros((2, 2, 2)))
    assert e.value.kind == "degenerate_input_error"
    bad = np.ones((2, 2, 2))
    bad[0, 0, 0] = np.nan
    with pytest.raises(ppo.OracleError) as e:
        ppo.svd(bad[:, :, 0])
    assert e.value.kind == "numeric_error"


def test_oracle_vs_numpy_tsvdq():
    a = ppo.random_tensor(20, 15, 12, 3)
    q = ppo.random_orthogonal_q(12, 5, 4)
    U, S, V = ppo.tsvdq(a, q, 4)
    ah = np.einsum("ijk,kl->ijl", a, q)
    for i in range(5):
        s = np.linalg.svd(ah[:, :, i], compute_uv=False)
        np.testing.assert_allclose(S[:, i], s[:4], rtol=1e-13)
    rec = ppo.tsvdq_reconstruct(U, S, V, q)
    want = np.zeros_like(a)
    for i in range(5):
        u, s, vt = np.linalg.svd(ah[:, :, i])
        want += np.einsum("ij,k->ijk", (u[:, :4] * s[:4]) @ vt[:4], q[:, i])
    assert np.linalg.norm(rec - want) <= 1e-12 * np.linalg.norm(a)


def test_random_orthogonal_deterministic():
    # tests/test_transforms.cpp:27-40
    t = ppo.random_orthogonal_q(8, 5, 1)
    assert np.abs(t.T @ t - np.eye(5)).max() <= 1e-10
    assert np.array_equal(t, ppo.random_orthogonal_q(8, 5, 1))
    assert np.abs(t - ppo.random_orthogonal_q(8, 5, 2)).max() > 1e-6


# ---------------------------------------------------------------- tsvdq2
def test_tsvdq2_gamma_one_keeps_numerical_rank():
    # tests/test_decompositions.cpp:126-146
    a = ppo.random_tensor(4, 5, 6, 44)
    q = ppo.dct_q(6, 4)
    U, S, V, mr = ppo.tsvdq2(a, q, 1.0)
    sp = ppo.slice_spectra(a, q)
    for i in range(4):
        assert mr[i] == int(np.sum(sp[:, i] > 1e-12 * sp[0, i]))
    tot, ey, pr = ppo.tsvdq2_error(a, U, S, V, q, mr)
    nrm = np.linalg.norm(a)
    assert abs(tot - ppo.projection_error(a, q)) <= 1e-10 * nrm
    assert ey <= 1e-10 * nrm
    for g in (0.0, 1.5, -0.1):
        with pytest.raises(ValueError):
            ppo.tsvdq2(a, q, g)


def test_tsvdq2_tie_break_counterexample():
    # tests/test_decompositions.cpp:148-160; verify.cpp:205-211
    a = counterexample()
    q = np.eye(2)
    U, S, V, mr = ppo.tsvdq2(a, q, 0.5)
    assert list(mr) == [2, 0]
    tot, _, _ = ppo.tsvdq2_error(a, U, S, V, q, mr)
    assert abs(tot * tot - 2.0) <= 1e-12
    # padded stacks: the dropped slice is all zeros
    assert not S[:, 1].any() and not U[:, :, 1].any() and not V[:, :, 1].any()


def test_tsvdq2_exact_rank_reproduces_tsvdq():
    # tests/test_decompositions.cpp:162-177
    q = ppo.dct_q(5, 3)
    hat = np.zeros((4, 4, 3), order="F")
    for s in range(3):
        hat[:, :, s] = ppo.random_matrix(4, 2, 300 + s) @ ppo.random_matrix(4, 2, 400 + s).T
    a = ppo.mode3_product(hat, q)
    U2, S2, V2, mr = ppo.tsvdq2(a, q, 1.0)
    assert list(mr) == [2, 2, 2]
    U1, S1, V1 = ppo.tsvdq(a, q, 2)
    nrm = np.linalg.norm(a)
    r2 = ppo.tsvdq_reconstruct(U2, S2, V2, q, 5)
    r1 = ppo.tsvdq_reconstruct(U1, S1, V1, q, 5)
    assert np.linalg.norm(r2 - r1) <= 1e-12 * nrm
    assert abs(ppo.tsvdq2_error(a, U2, S2, V2, q, mr)[0] - ppo.tsvdq_error(a, U1, S1, V1, q)[0]) \
        <= 1e-12 * nrm


def test_tsvdq2_full_transform_lossless():
    # tests/test_decompositions.cpp:179-188
    a = ppo.random_tensor(3, 4, 4, 46)
    q = ppo.dct_q(4, 4)
    U, S, V, mr = ppo.tsvdq2(a, q, 1.0)
    tot, ey, pr = ppo.tsvdq2_error(a, U, S, V, q, mr)
    nrm = np.linalg.norm(a)
    assert tot <= 1e-10 * nrm and ey <= 1e-10 * nrm and pr <= 1e-10 * nrm


def test_tsvdq2_error_decomposition_and_selection_rule():
    # tests/test_decompositions.cpp:190-205, plus the selection restated in numpy
    for i in range(10):
        a = ppo.random_tensor(4, 3, 5, 470 + i)
        q = ppo.random_orthogonal_q(5, 3, 100 + i)
        U, S, V, mr = ppo.tsvdq2(a, q, 0.8)
        tot, ey, pr = ppo.tsvdq2_error(a, U, S, V, q, mr)
        assert abs(tot ** 2 - (ey ** 2 + pr ** 2)) <= 1e-10 * tot ** 2
        direct = np.linalg.norm(a - ppo.tsvdq_reconstruct(U, S, V, q, 5))
        assert abs(tot - direct) <= 1e-10 * np.linalg.norm(a)
        # independent restatement of decompositions.cpp:131-176 on LAPACK spectra
        ah = np.einsum("ijk,kp->ijp", a, q)
        sp = np.stack([np.linalg.svd(ah[:, :, s], compute_uv=False) for s in range(3)], axis=1)
        pool = [(-sp[j, s], s, j) for s in range(3) for j in range(sp.shape[0])
                if sp[j, s] > 1e-12 * sp[0].max()]
        pool.sort()
        cum = np.cumsum([v * v for v, _, _ in pool])
        K = min(int(np.searchsorted(cum, 0.8 * cum[-1], side="left")) + 1, len(pool))
        want = np.zeros(3, dtype=int)
        for _, s, _ in pool[:K]:
            want[s] += 1
        assert list(mr) == list(want)


# --------------------------------------------------- star-M and baselines
def test_star_m_kats():
    # tests/test_star_products.cpp:34-55
    a, b = tube([2, 4, 6, 8]), tube([1, -1, 1, 0])
    np.testing.assert_allclose(ppo.star_m_product(a, b, ppo.haar_q(4, 4).T).ravel(), [2, 4, 3, 8],
                               atol=1e-12)
    np.testing.assert_allclose(ppo.star_m_product(tube([1, 2, 3]), tube([4, -5, 0.5]), np.eye(3)).ravel(),
                               [4, -10, 1.5], atol=1e-14)
    A = ppo.random_tensor(2, 3, 4, 31)
    B = ppo.random_tensor(3, 2, 4, 32)
    M = ppo.random_matrix(4, 4, 33)
    fast = ppo.star_m_product(A, B, M)
    slow = ppo.star_m_by_tubes(A, B, M)
    assert np.linalg.norm(fast - slow) <= 1e-12 * np.linalg.norm(fast)
    sing = np.zeros((2, 2))
    sing[0, 0] = 1.0
    with pytest.raises(ValueError):
        ppo.star_m_product(tube([1, 2]), tube([1, 2]), sing)


def test_mode_unfold_and_mode_product_kats():
    """test_tensor.cpp:87-99 (unfold pins) and :123-134 (mode products vs the
    unfolding identity (A x_m M)_(m) = M A_(m))."""
    A = counterexample()
    assert np.array_equal(ppo.mode_unfold(A, 3), A.reshape(4, 2, order="F").T)
    I = np.zeros((2, 2, 2), order="F")
    I[:, :, 0] = I[:, :, 1] = np.eye(2)
    assert np.array_equal(ppo.mode_unfold(I, 1), np.array([[1, 0, 1, 0], [0, 1, 0, 1.0]]))
    assert not ppo.mode_unfold(np.zeros((3, 2, 2)), 2).any()
    a = ppo.random_tensor(3, 4, 5, 7)
    for mode, ext in ((1, 3), (2, 4), (3, 5)):
        m = ppo.random_matrix(6, ext, 20 + mode)
        got = ppo.mode_product(a, m, mode)
        assert np.abs(ppo.mode_unfold(got, mode) - m @ ppo.mode_unfold(a, mode)).max() <= 1e-13
    assert np.abs(ppo.mode_product(a, m, 3) - ppo.mode3_product(a, m)).max() <= 1e-13
    with pytest.raises(ValueError):
        ppo.mode_product(a, m, 4)


def test_hosvd_kats():
    # tests/test_decompositions.cpp:203-232
    A = ppo.random_tensor(4, 3, 5, 48)
    core, U1, U2, U3 = ppo.hosvd(A, 4, 3, 5)
    assert np.linalg.norm(A - ppo.hosvd_reconstruct(core, U1, U2, U3)) <= 1e-10 * np.linalg.norm(A)
    for U, n in ((U1, 4), (U2, 3), (U3, 5)):
        assert np.linalg.norm(U.T @ U - np.eye(n)) <= 1e-10 * n
    x, y, z = ppo.random_matrix(4, 1, 1), ppo.random_matrix(3, 1, 2), ppo.random_matrix(5, 1, 3)
    R = np.einsum("i,j,k->ijk", x[:, 0], y[:, 0], z[:, 0])
    f = ppo.hosvd(R, 1, 1, 1)
    assert np.linalg.norm(R - ppo.hosvd_reconstruct(*f)) <= 1e-10 * np.linalg.norm(R)
    C = counterexample()
    err = np.linalg.norm(C - ppo.hosvd_reconstruct(*ppo.hosvd(C, 2, 2, 1)))
    assert abs(err * err - 2.0) <= 1e-12
    for bad in ((0, 1, 1), (1, 4, 1)):
        with pytest.raises(ValueError):
            ppo.hosvd(A, *bad)


def test_matrix_svd_baseline_kats():
    # tests/test_decompositions.cpp:234-255
    A = ppo.random_tensor(3, 4, 5, 49)
    assert ppo.matrix_svd_baseline(A, 4)[3] <= 1e-10 * np.linalg.norm(A)
    U, s, V, err = ppo.matrix_svd_baseline(counterexample(), 1)
    assert s.shape == (1,) and abs(s[0] - SQ2) <= 1e-12 and abs(err * err - 2.0) <= 1e-12
    assert ppo.matrix_svd_baseline(np.zeros((2, 3, 2)), 2)[3] == 0.0
    for k in (0, 5):
        with pytest.raises(ValueError):
            ppo.matrix_svd_baseline(A, k)


def test_lapack_baseline_matches_oracle():
    """oracle/baseline.py (the CPU-baseline restatement of the compress chain
    on LAPACK, bench.py's cpu_baseline / --impl reference for cfg5) is pinned
    to the C oracle: same basis (captured energies, sign rule), same slice
    singular values with a shared basis, same relative error."""
    from oracle import baseline
    from paper_2409_19402_b200 import synth
    a = synth.cp_tensor(24, 20, 16, rank=3, noise=1e-2, seed=2)
    q, U, S, V, re = baseline.compress(a, 6, 3)
    qo, _, _ = ppo.data_dependent_q(a, 6)
    T = a.reshape(-1, 16, order="F")
    np.testing.assert_allclose(np.sum((T @ q) ** 2, axis=0), np.sum((T @ qo) ** 2, axis=0), rtol=1e-10)
    np.testing.assert_allclose(np.abs(q.T @ qo), np.eye(6), atol=1e-8)  # well-separated spectrum
    Uo, So, Vo = ppo.tsvdq(a, q, 3)
    np.testing.assert_allclose(S, So, rtol=1e-10)
    re_o = ppo.relative_error(a, ppo.tsvdq_reconstruct(Uo, So, Vo, q))
    assert abs(re - re_o) <= 1e-10 * re_o
    sec, det = baseline.compress_timed(lambda w: np.asfortranarray(a[:, :w, :]), 24, 20, 16, 6, 3, 5,
                                       lambda i: np.asfortranarray(a[:, :, i]))
    assert sec > 0 and det["n_linear_scale"] == 4.0
