"""Time the top-p eigensolver's tridiagonal reduction (stage timer
eig.tridiag) for one symmetric n x n matrix.

  python tools/trd_time.py n p [reps]
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2409_19402_b200 import _lib  # noqa: E402

n, p = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rng = np.random.default_rng(0)
X = rng.standard_normal((2 * n, n))
G = X.T @ X
L = _lib.lib()
g = torch.tensor(np.asfortranarray(G).ravel(order="F"), device="cuda")
Q = torch.empty((p, n), dtype=torch.float64, device="cuda")
S = torch.empty(p, dtype=torch.float64, device="cuda")
args = (C.c_void_p(g.data_ptr()), n, p, C.c_void_p(Q.data_ptr()), C.c_void_p(S.data_ptr()), 1)
assert L.ppc_sym_eig_top(*args) == 0
torch.cuda.synchronize()
buf = C.create_string_buffer(1 << 16)
L.ppc_timing_report(buf, len(buf), 1)
L.ppc_timing_enable(1)
for _ in range(reps):
    L.ppc_sym_eig_top(*args)
torch.cuda.synchronize()
L.ppc_timing_report(buf, len(buf), 1)
d = json.loads(buf.value.decode())
w = np.linalg.eigvalsh(G)[::-1][:p]
err = np.max(np.abs(S.cpu().numpy() ** 2 - w)) / w[0]
print(f"n={n} "
      f"tridiag {d['eig.tridiag']['ms'] / reps:.3f} ms  per step {1e3 * d['eig.tridiag']['ms'] / reps / (n - 2):.2f} us  "
      f"eig err {err:.1e}", flush=True)
