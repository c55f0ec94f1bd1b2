"""Ozaki Gram on exactly representable data (small integers, and integers
times one power of two per column): the digit products are exact, so the
result must equal the exact Gram bit for bit."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2409_19402_b200 import _lib  # noqa: E402

L = _lib.lib()
rows, n3 = 1 << 20, 512
rng = np.random.default_rng(0)
for kind in ("int", "wide"):
    if kind == "int":
        T = rng.integers(-8, 9, size=(rows, n3)).astype(np.float64)
    else:
        T = rng.integers(-(1 << 20), 1 << 20, size=(rows, n3)).astype(np.float64) * 2.0 ** -30
    Tf = np.asfortranarray(T)
    Td = torch.from_numpy(Tf.T.copy()).cuda().T  # Fortran layout on device
    c, ch = C.c_int64(), C.c_int64()
    assert L.ppc_gram_plan(rows, n3, C.byref(c), C.byref(ch)) == 0
    parts = torch.zeros(c.value * n3 * n3, dtype=torch.float64, device="cuda")
    rc = L.ppc_gram_partials(C.c_void_p(Td.data_ptr()), rows, rows, n3, ch.value, c.value,
                             C.c_void_p(parts.data_ptr()), 1)
    assert rc == 0, L.ppc_last_error()
    P = parts.view(c.value, n3, n3).sum(0).cpu().numpy()
    G = Tf.T @ Tf  # exact for these values
    d = np.abs(P - G)
    print(kind, "chunks", c.value, "chunk", ch.value, "max rel diff", d.max() / np.abs(G).max(),
          "exact entries", float(np.mean(d == 0)))
