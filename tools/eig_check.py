"""Top-p eigensolver (ppc_sym_eig_top) on cfg5-like and adversarial Grams:
eigenvalues vs numpy eigh, orthonormality, residuals, captured energy, time.
PPC_TRIDIAG_EIG=0 switches the direct solver off (subspace iteration).

  python tools/eig_check.py
"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2409_19402_b200 import _lib  # noqa: E402

L = _lib.lib()


def gram_case(kind, n, seed=0):
    rng = np.random.default_rng(seed)
    if kind == "cp":  # rank-50 spikes over a Marchenko-Pastur noise plateau (cfg5 shape)
        F = rng.standard_normal((n, 50)) * np.sqrt(np.logspace(9.8, 6, 50))
        Nn = rng.standard_normal((n, 4 * n))
        G = F @ F.T + 4.2 / (4 * n) * (Nn @ Nn.T)
    elif kind == "lowrank":  # rank 30: zero-eigenvalue cluster inside the top p
        F = rng.standard_normal((n, 30))
        G = F @ F.T
    elif kind == "cluster":  # exactly repeated eigenvalues
        Qr, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = np.concatenate([np.full(40, 5.0), np.full(40, 3.0), np.linspace(1, 0, n - 80)])
        G = (Qr * lam) @ Qr.T
    else:
        X = rng.standard_normal((4 * n, n))
        G = X.T @ X
    return 0.5 * (G + G.T)


def run(G, p, reps=5):
    n = G.shape[0]
    g = torch.tensor(np.asfortranarray(G).ravel(order="F"), device="cuda")
    Qd = torch.empty((p, n), dtype=torch.float64, device="cuda")
    Sd = torch.empty(p, dtype=torch.float64, device="cuda")
    args = (C.c_void_p(g.data_ptr()), n, p, C.c_void_p(Qd.data_ptr()), C.c_void_p(Sd.data_ptr()), 1)
    rc = L.ppc_sym_eig_top(*args)
    assert rc == 0, L.ppc_last_error()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        L.ppc_sym_eig_top(*args)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    return Qd.cpu().numpy().T, Sd.cpu().numpy() ** 2, ms


for kind, n, p in [("cp", 1024, 128), ("cp", 1024, 64), ("lowrank", 512, 48), ("cluster", 300, 100),
                   ("gauss", 224, 32), ("gauss", 200, 20), ("cp", 1536, 160)]:
    G = gram_case(kind, n)
    w, U = np.linalg.eigh(G)
    w, U = w[::-1], U[:, ::-1]
    Q, lam, ms = run(G, p)
    l1 = w[0]
    ev = np.max(np.abs(lam - w[:p])) / l1
    orth = np.max(np.abs(Q.T @ Q - np.eye(p)))
    res = np.max(np.linalg.norm(G @ Q - Q * lam, axis=0)) / l1
    cap = abs(np.trace(Q.T @ G @ Q) - w[:p].sum()) / w[:p].sum()
    print(f"{kind:8s} n={n:5d} p={p:4d}  eig {ev:.2e}  orth {orth:.2e}  res {res:.2e}  energy {cap:.2e}  {ms:7.2f} ms",
          flush=True)
