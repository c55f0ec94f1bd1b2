"""Standalone probe: Gram SYRK (data-driven Q path) at a given shape on cuda:0,
timed with CUDA events (used for ncu captures of the SYRK kernel alone)."""
import ctypes as C
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_19402_b200 as pp
from paper_2409_19402_b200 import _lib
n1, n2, n3, p = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (2048, 2048, 1024, 128)))
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
L = _lib.lib()
A = torch.randn(n3, n2, n1, dtype=torch.float64, device="cuda").permute(2, 1, 0)
Q = pp.empty_device((n3, p))
comp = C.c_int()
s = torch.cuda.current_stream()
L.ppc_set_stream(C.c_void_p(s.cuda_stream))
L.ppc_timing_enable(1)
for _ in range(reps):
    rc = L.ppc_data_dependent_q(C.c_void_p(A.data_ptr()), n1, n2, n3, p, C.c_void_p(Q.data_ptr()), None, C.byref(comp), 1)
    assert rc == 0, L.ppc_last_error()
torch.cuda.synchronize()
buf = C.create_string_buffer(1 << 16)
L.ppc_timing_report(buf, len(buf), 1)
print(buf.value.decode())
