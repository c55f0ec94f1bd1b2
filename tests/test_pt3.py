"""PT3 container I/O through the engine's C-ABI (ppc_pt3_*), host mode (no GPU
needed): byte parity with the oracle's restatement of io.cpp:52-126 and the
reference's own io tests (tests/test_io.cpp:50-112)."""
import numpy as np
import pytest

from oracle import ppo
from paper_2409_19402_b200 import projprod as pp


def test_writer_bytes_match_reference_layout(tmp_path):
    a = ppo.random_tensor(4, 3, 5, 71)
    f = tmp_path / "a.pt3"
    pp.write_pt3(f, a)
    assert f.read_bytes() == ppo.pt3_bytes(a)
    m = ppo.random_matrix(3, 7, 5)
    pp.write_pt3_matrix(tmp_path / "m.pt3", m)
    assert (tmp_path / "m.pt3").read_bytes() == ppo.pt3_bytes(m)


def test_round_trip_bit_exact(tmp_path):
    # tests/test_io.cpp:50-61
    a = ppo.random_tensor(4, 3, 5, 71)
    f = tmp_path / "rt.pt3"
    pp.write_pt3(f, a)
    assert pp.pt3_shape(f) == (4, 3, 5)
    b = pp.read_pt3(f)
    assert b.shape == (4, 3, 5) and b.tobytes(order="F") == np.asfortranarray(a).tobytes(order="F")
    # oracle-written files read back identically
    g = tmp_path / "or.pt3"
    g.write_bytes(ppo.pt3_bytes(a))
    assert np.array_equal(pp.read_pt3(g), a)
    np.testing.assert_array_equal(ppo.pt3_parse(f.read_bytes()), a)


def test_matrix_container(tmp_path):
    # tests/test_io.cpp:63-71
    m = ppo.random_matrix(3, 7, 5)
    f = tmp_path / "m.pt3"
    pp.write_pt3_matrix(f, m)
    r = pp.read_pt3_matrix(f)
    assert r.shape == (3, 7) and np.abs(m - r).max() == 0.0
    pp.write_pt3(tmp_path / "t.pt3", ppo.random_tensor(2, 2, 3, 1))
    with pytest.raises(pp.FormatError):
        pp.read_pt3_matrix(tmp_path / "t.pt3")


def test_rejects_malformed_files(tmp_path):
    # tests/test_io.cpp:73-112
    a = ppo.random_tensor(2, 2, 2, 72)
    f = tmp_path / "bad.pt3"
    pp.write_pt3(f, a)
    good = f.read_bytes()

    def tampered(buf):
        f.write_bytes(bytes(buf))
        with pytest.raises(pp.FormatError):
            pp.read_pt3(f)
        with pytest.raises(ValueError):  # the oracle agrees
            ppo.pt3_parse(bytes(buf))

    for off, val in ((0, ord("X")), (4, 9), (8, 7), (9, 1)):
        b = bytearray(good)
        b[off] = val
        tampered(b)
    tampered(good[:-1])                       # truncated payload
    tampered(good + b"\0")                    # trailing garbage
    b = bytearray(good)
    b[12:20] = b"\xff" * 8                    # extent overflow
    tampered(b)
    b = bytearray(good)
    b[12:20] = b"\0" * 8                      # zero extent
    tampered(b)
    tampered(good[:20])                       # truncated header
    with pytest.raises(pp.FormatError):
        pp.read_pt3(str(f) + ".does-not-exist")


def test_destination_size_checked(tmp_path):
    import ctypes as C
    from paper_2409_19402_b200 import _lib
    f = tmp_path / "s.pt3"
    pp.write_pt3(f, ppo.random_tensor(2, 3, 4, 1))
    out = np.empty(23)
    assert _lib.lib().ppc_pt3_read(str(f).encode(), C.c_void_p(out.ctypes.data), 23, _lib.PPC_HOST) == 1


def test_factor_export_layout(tmp_path):
    # tools/main.cpp:211-217: U (n1,k,p), S (k,1,p), V (n2,k,p), Q (n3,p,1)
    n1, n2, n3, k, p = 5, 4, 6, 2, 3
    rng = np.random.default_rng(0)
    q = ppo.dct_q(n3, p)
    f = pp.TsvdqFactors(rng.standard_normal((n1, k, p)), rng.standard_normal((k, p)),
                        rng.standard_normal((n2, k, p)), pp.Transform.custom(q), k, n1, n2)
    pre = str(tmp_path / "fac")
    pp.write_tsvdq_factors(pre, f)
    assert pp.pt3_shape(pre + ".U.pt3") == (n1, k, p)
    assert pp.pt3_shape(pre + ".S.pt3") == (k, 1, p)
    assert pp.pt3_shape(pre + ".V.pt3") == (n2, k, p)
    assert pp.pt3_shape(pre + ".Q.pt3") == (n3, p, 1)
    assert np.array_equal(pp.read_pt3(pre + ".S.pt3")[:, 0, :], f.s)
    assert np.array_equal(pp.read_pt3_matrix(pre + ".Q.pt3"), q)
