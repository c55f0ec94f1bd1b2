"""One cfg5-shaped ppc_tsvdq_compress after `--warm` untimed calls, for ncu
launch lists and debug traces (PPC_SUBSPACE_DEBUG / PPC_JACOBI_DEBUG) that
cover exactly one call.  Prints the stage timers of the last call.

  python tools/prof_compress.py [--shape 2048 2048 1024] [--p 128] [--k 32] [--warm 1]
"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--shape", type=int, nargs=3, default=[2048, 2048, 1024])
ap.add_argument("--p", type=int, default=128)
ap.add_argument("--k", type=int, default=32)
ap.add_argument("--warm", type=int, default=1)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--per-call", action="store_true", help="stage timers of every call (slow calls only)")
ap.add_argument("--empty-cache", action="store_true", help="return torch's cached blocks after building A")
args = ap.parse_args()

import torch  # noqa: E402
import paper_2409_19402_b200 as pp  # noqa: E402
from paper_2409_19402_b200 import _lib, synth  # noqa: E402

L = _lib.lib()
n1, n2, n3 = args.shape
p, k = args.p, args.k
A = synth.cp_tensor_device(n1, n2, n3, rank=50, noise=1e-3, seed=0)
if args.empty_cache:
    torch.cuda.empty_cache()
Q = pp.empty_device((n3, p))
U = pp.empty_device((n1, k, p))
S = pp.empty_device((k, p))
V = pp.empty_device((n2, k, p))
torch.cuda.synchronize()


def call():
    re = C.c_double()
    rc = L.ppc_tsvdq_compress(C.c_void_p(A.data_ptr()), n1, n2, n3, p, k, C.c_void_p(Q.data_ptr()), None,
                              C.c_void_p(U.data_ptr()), C.c_void_p(S.data_ptr()), C.c_void_p(V.data_ptr()),
                              C.byref(re), 1)
    if rc:
        raise RuntimeError(L.ppc_last_error().decode())
    return re.value


for _ in range(args.warm):
    call()
torch.cuda.synchronize()
fr, tot = torch.cuda.mem_get_info()
print(f"device memory: free {fr / 1e9:.1f} GB of {tot / 1e9:.1f}; torch reserved {torch.cuda.memory_reserved() / 1e9:.1f} GB",
      flush=True)
buf = C.create_string_buffer(1 << 16)
L.ppc_timing_report(buf, len(buf), 1)
L.ppc_timing_enable(1)
for _ in range(args.reps):
    t0 = time.perf_counter()
    re = call()
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t0)
    print(f"compress {ms:.1f} ms  RE {re:.12e}", flush=True)
    if args.per_call:
        L.ppc_timing_report(buf, len(buf), 1)
        if ms > 200:
            import json
            d = json.loads(buf.value.decode())
            print("SLOW", {k: round(v["ms"], 2) for k, v in d.items()}, flush=True)
L.ppc_timing_enable(0)
L.ppc_timing_report(buf, len(buf), 1)
print(buf.value.decode())
