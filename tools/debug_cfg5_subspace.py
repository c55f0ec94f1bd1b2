"""One cfg5 compress with PPC_SUBSPACE_DEBUG=1: per-iteration locking of the
slice-SVD subspace iteration (stderr)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PPC_SUBSPACE_DEBUG", "1")
import torch  # noqa: E402
import paper_2409_19402_b200 as pp  # noqa: E402
from paper_2409_19402_b200 import _lib, synth  # noqa: E402

n1, n2, n3, p, k = [int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (2048, 2048, 1024, 128, 32))]
L = _lib.lib()
A = synth.cp_tensor_device(n1, n2, n3, rank=50, noise=1e-3, seed=0)
Q = pp.empty_device((n3, p))
U = pp.empty_device((n1, k, p))
S = pp.empty_device((k, p))
V = pp.empty_device((n2, k, p))
re = C.c_double()
L.ppc_timing_enable(1)
rc = L.ppc_tsvdq_compress(C.c_void_p(A.data_ptr()), n1, n2, n3, p, k, C.c_void_p(Q.data_ptr()), None,
                          C.c_void_p(U.data_ptr()), C.c_void_p(S.data_ptr()), C.c_void_p(V.data_ptr()),
                          C.byref(re), 1)
assert rc == 0, L.ppc_last_error()
buf = C.create_string_buffer(1 << 16)
L.ppc_timing_report(buf, len(buf), 1)
print("re", re.value)
print(buf.value.decode())
s = pp.to_host(S)
print("s[0,:]", s[0, ::8])
print("s[k-1,:]", s[k - 1, ::8])
