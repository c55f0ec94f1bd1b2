"""cfg4 star-Q product through host buffers with PPC_STARQ_TRACE=1: the
timeline of the host pipeline's copies and compute (stderr)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PPC_STARQ_TRACE", "1")
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2409_19402_b200 import _lib  # noqa: E402

L = _lib.lib()
wl = bench.make_workload("cfg4")
wl.e2e_setup()
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    wl.e2e_step(L)
    torch.cuda.synchronize()
    print(f"e2e step {it}: {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr, flush=True)
