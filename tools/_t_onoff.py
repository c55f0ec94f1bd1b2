import sys, time, ctypes as C
sys.path.insert(0, '.')
import torch
import paper_2409_19402_b200 as pp
from paper_2409_19402_b200 import _lib, synth
L = _lib.lib()
n1 = n2 = 2048; n3 = 1024; p = 128; k = 32
A = synth.cp_tensor_device(n1, n2, n3, rank=50, noise=1e-3, seed=0)
Q = pp.empty_device((n3, p)); U = pp.empty_device((n1, k, p)); S = pp.empty_device((k, p)); V = pp.empty_device((n2, k, p))
def call():
    re = C.c_double()
    rc = L.ppc_tsvdq_compress(C.c_void_p(A.data_ptr()), n1, n2, n3, p, k, C.c_void_p(Q.data_ptr()), None,
                              C.c_void_p(U.data_ptr()), C.c_void_p(S.data_ptr()), C.c_void_p(V.data_ptr()), C.byref(re), 1)
    assert rc == 0
for _ in range(2): call()
torch.cuda.synchronize()
for on in (0, 1, 0, 1):
    L.ppc_timing_enable(on)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter(); call(); torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
    print("timing", on, " ".join(f"{t:.1f}" for t in ts), flush=True)
