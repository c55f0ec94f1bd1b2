"""Exact reference for the Ozaki SYRK: replicate the split (balanced 8-bit
digits, 6 digits) in numpy with exact integer arithmetic, form the 21
digit-pair level sums with Python integers and compare with the kernel."""
import ctypes as C
import os
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2409_19402_b200 import _lib, synth  # noqa: E402

L = _lib.lib()
rows, n = 4096, 128
A = synth.cp_tensor_device(64, 64, n, rank=50, noise=1e-3, seed=3).reshape(rows, n)  # Fortran (rows, n)
G = torch.empty(n * n, dtype=torch.float64, device="cuda")
rc = L.ppc_ozaki_syrk_batched(C.c_void_p(A.data_ptr()), rows, rows * n, rows, n, 1, C.c_void_p(G.data_ptr()))
assert rc == 0, L.ppc_last_error()
torch.cuda.synchronize()
Gk = G.view(n, n).T.cpu().numpy()  # column-major -> (row, col)
X = A.cpu().numpy()  # (rows, n)


def digits(col):
    mx = np.abs(col).max()
    e = int(np.frexp(mx)[1]) - 1 + 2  # ilogb(mx) + 2
    # y = rint(x * 2^(47-e)) (integer), value 128 x / sigma ~ y * 2^-40
    Y = np.array([int(round(v * 2.0 ** (47 - e))) for v in col], dtype=object)  # exact (|v 2^k| < 2^53)
    c = sum(128 << (8 * (5 - s)) for s in range(1, 6))  # offset in units of 2^-40
    U = Y + c
    d = []
    d1 = [u >> 40 for u in U]  # floor division (python >> floors for negatives)
    rem = [u - (q << 40) for u, q in zip(U, d1)]
    d.append(np.array(d1, dtype=object))
    for s in range(1, 6):
        sh = 40 - 8 * s
        q = [r >> sh for r in rem]
        rem = [r - (x << sh) for r, x in zip(rem, q)]
        d.append(np.array([x - 128 for x in q], dtype=object))
    return e, d


info = [digits(X[:, j]) for j in range(n)]
worst = 0.0
mism = 0
for a in range(0, n, 17):
    for b in range(a, n, 13):
        ea, da = info[a]
        eb, db = info[b]
        tot = Fraction(0)
        for s in range(6):
            for t in range(6):
                if s + t + 2 <= 7:
                    q = int(np.dot(da[s], db[t]))
                    tot += Fraction(q, 1 << (14 + 8 * (s + t)))
        ref = float(tot * Fraction(2) ** (ea + eb))
        got = Gk[a, b]
        exact = float(np.dot(X[:, a], X[:, b]))
        if got != ref:
            mism += 1
        worst = max(worst, abs(got - ref) / max(abs(ref), 1e-300))
        print(a, b, "kernel-vs-digits", abs(got - ref) / max(abs(ref), 1e-300), "digits-vs-fp64", abs(ref - exact) / abs(exact))
print("mismatches", mism, "worst", worst)
