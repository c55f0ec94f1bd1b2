"""cfg5 compress through host buffers (the bench's e2e call) with the stage
timers on, next to a plain pinned H2D of the same 32 GiB: where the e2e time
goes beyond PCIe."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2409_19402_b200 import _lib, synth  # noqa: E402

L = _lib.lib()
n1, n2, n3, p, k = 2048, 2048, 1024, 128, 32
A = synth.cp_tensor_device(n1, n2, n3, rank=50, noise=1e-3, seed=0)
hA = torch.empty(n1 * n2 * n3, dtype=torch.float64).pin_memory()
hA.copy_(A.permute(2, 1, 0).reshape(-1))
del A
torch.cuda.empty_cache()
d = torch.empty(n1 * n2 * n3, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter()
    d.copy_(hA, non_blocking=True)
    torch.cuda.synchronize()
    print(f"plain H2D {1e3 * (time.perf_counter() - t0):.1f} ms ({hA.numel() * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s)")
del d
torch.cuda.empty_cache()
hQ, hU, hS, hV = (torch.empty(n, dtype=torch.float64).pin_memory() for n in (n3 * p, n1 * k * p, k * p, n2 * k * p))
buf = C.create_string_buffer(1 << 16)


def call():
    re = C.c_double()
    rc = L.ppc_tsvdq_compress(C.c_void_p(hA.data_ptr()), n1, n2, n3, p, k, C.c_void_p(hQ.data_ptr()), None,
                              C.c_void_p(hU.data_ptr()), C.c_void_p(hS.data_ptr()), C.c_void_p(hV.data_ptr()),
                              C.byref(re), 0)
    assert rc == 0, L.ppc_last_error()
    return re.value


call()
L.ppc_timing_report(buf, len(buf), 1)
for _ in range(2):
    L.ppc_timing_enable(1)
    t0 = time.perf_counter()
    re = call()
    print(f"e2e compress {1e3 * (time.perf_counter() - t0):.1f} ms RE {re:.12e}")
    L.ppc_timing_enable(0)
    L.ppc_timing_report(buf, len(buf), 1)
    print(buf.value.decode())
