"""Time the one-CTA Jacobi eigensolver (logged / smem paths) on one b x b PSD
matrix, as in the Rayleigh-Ritz step of the eigenbasis (batch 1)."""
import sys
import time

import os
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2409_19402_b200 import _lib

L = _lib.lib()
for b, kind in [(160, "rand"), (160, "neardiag"), (110, "rand"), (110, "neardiag"), (64, "rand")]:
    g = torch.Generator().manual_seed(0)
    if kind == "rand":
        X = torch.randn(b, b, dtype=torch.float64, generator=g)
        lam = torch.logspace(0, -6, b, dtype=torch.float64)
        Q, _ = torch.linalg.qr(X)
        H = (Q * lam) @ Q.T
    else:
        lam = torch.logspace(0, -6, b, dtype=torch.float64)
        E = 1e-4 * torch.randn(b, b, dtype=torch.float64, generator=g)
        H = torch.diag(lam) + (E + E.T) * torch.sqrt(lam[:, None] * lam[None, :])
    H = H.cuda().contiguous()
    p = b - 8
    Qo = torch.empty(b, p, dtype=torch.float64, device="cuda")
    so = torch.empty(p, dtype=torch.float64, device="cuda")
    for _ in range(3):
        rc = L.ppc_sym_eig_top(H.data_ptr(), b, p, Qo.data_ptr(), so.data_ptr(), 1)
        assert rc == 0, L.ppc_last_error()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 10
    for _ in range(n):
        L.ppc_sym_eig_top(H.data_ptr(), b, p, Qo.data_ptr(), so.data_ptr(), 1)
    e1.record()
    torch.cuda.synchronize()
    ev = torch.linalg.eigvalsh(H.cpu())
    err = (torch.sort(ev, descending=True).values[:p] - so.cpu() ** 2).abs().max().item()
    print(f"b={b} {kind}: {e0.elapsed_time(e1)/n:.3f} ms/eig  max|lam err|={err:.2e}", flush=True)
