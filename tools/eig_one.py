"""One ppc_sym_eig_top call on a cfg5-like Gram (n=1024, p=128), for ncu."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2409_19402_b200 import _lib  # noqa: E402

n, p = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (1024, 128)))
rng = np.random.default_rng(0)
F = rng.standard_normal((n, 50)) * np.sqrt(np.logspace(9.8, 6, 50))
Nn = rng.standard_normal((n, 4 * n))
G = F @ F.T + 4.2 / (4 * n) * (Nn @ Nn.T)
G = 0.5 * (G + G.T)
L = _lib.lib()
g = torch.tensor(np.asfortranarray(G).ravel(order="F"), device="cuda")
Q = torch.empty((p, n), dtype=torch.float64, device="cuda")
S = torch.empty(p, dtype=torch.float64, device="cuda")
rc = L.ppc_sym_eig_top(C.c_void_p(g.data_ptr()), n, p, C.c_void_p(Q.data_ptr()), C.c_void_p(S.data_ptr()), 1)
torch.cuda.synchronize()
print("rc", rc)
