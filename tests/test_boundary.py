"""The C-ABI boundary: libppc.so loads, exports every symbol include/ppc.h
declares, host-side builders work without a GPU, and compute calls fail
loudly (no CPU fallback) when no device is visible. CPU only."""
import ctypes as C
import subprocess

import numpy as np
import pytest

from oracle import ppo
from paper_2409_19402_b200 import _lib

from conftest import gpu_available


def test_library_exports_every_header_symbol():
    syms = _lib.exported_symbols_from_header()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    L = _lib.lib()
    for s in syms:
        assert getattr(L, s) is not None
    assert L.ppc_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "DMMA.8x8x4" in sass  # FP64 tensor-core path


@pytest.mark.skipif(gpu_available(), reason="checks the no-device behaviour")
def test_no_cpu_fallback():
    import paper_2409_19402_b200 as pp
    a = np.ones((2, 2, 4))
    with pytest.raises(pp.EngineError, match="no CPU path"):
        pp.star_q(a, a, pp.Transform("dct", 4, 2))
    L = _lib.lib()
    out = C.c_double()
    rc = L.ppc_frobenius_norm(C.c_void_p(a.ctypes.data), a.size, C.byref(out), 0)
    assert rc == 8  # PPC_NO_DEVICE


def test_host_builders_match_oracle():
    import paper_2409_19402_b200 as pp
    assert np.abs(pp.Transform("dct", 17, 5).q - ppo.dct_q(17, 5)).max() <= 1e-15
    assert np.abs(pp.Transform("random", 32, 8, seed=1).q - ppo.random_orthogonal_q(32, 8, 1)).max() <= 1e-13
    assert np.array_equal(pp.Transform("haar", 4, 3).q, ppo.haar_q(4, 3))
    assert np.array_equal(pp.Transform("identity", 5, 2).q, np.eye(5)[:, :2])
    with pytest.raises(pp.ArgumentError):
        pp.Transform("identity", 4, 9)
    with pytest.raises(pp.ArgumentError):
        pp.Transform("haar", 3, 2)
    with pytest.raises(pp.DegenerateInputError):
        pp.Transform.custom(np.ones((4, 2)))
    with pytest.raises(pp.ArgumentError):
        pp.Transform.custom(np.eye(4)[:, :2], 0.0)
    with pytest.raises(pp.ArgumentError):
        pp.Transform("data", 4, 2)


def test_fp64_only_switch_without_gpu():
    """The arithmetic switch (ppc_set_ozaki / projprod.set_fp64_only) is host
    state: it works, and round-trips, without a device."""
    import paper_2409_19402_b200 as pp
    was = pp.fp64_only()
    try:
        pp.set_fp64_only(True)
        assert pp.fp64_only()
        pp.set_fp64_only(False)
        assert not pp.fp64_only()
    finally:
        pp.set_fp64_only(was)
    assert _lib.lib().ppc_set_ozaki(2) == 3  # PPC_ARGUMENT
