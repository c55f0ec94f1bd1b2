"""Ozaki INT8 Gram vs the FP64 DMMA Gram through ppc_gram_partials.
Run once with PPC_OZAKI=0 and once without; the second run compares."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2409_19402_b200 import _lib, synth  # noqa: E402

L = _lib.lib()
tag = "dmma" if os.environ.get("PPC_OZAKI") == "0" else "ozaki"
out = {}
for rows, n3, kind in ((1 << 18, 256, "gauss"), (1 << 20, 512, "cp"), (1 << 22, 1024, "cp")):
    if kind == "gauss":
        T = synth.gaussian_device(rows, 1, n3, 3, 1).reshape(rows, n3)
    else:
        T = synth.cp_tensor_device(1 << (rows.bit_length() // 2), rows >> (rows.bit_length() // 2), n3,
                                   rank=50, noise=1e-3, seed=1).reshape(rows, n3)
    c, ch = C.c_int64(), C.c_int64()
    assert L.ppc_gram_plan(rows, n3, C.byref(c), C.byref(ch)) == 0
    parts = torch.empty(c.value * n3 * n3, dtype=torch.float64, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = L.ppc_gram_partials(C.c_void_p(T.data_ptr()), rows, rows, n3, ch.value, c.value,
                                 C.c_void_p(parts.data_ptr()), 1)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        assert rc == 0, L.ppc_last_error()
    G = parts.view(c.value, n3, n3).sum(0).cpu().numpy()
    out[(rows, n3)] = G
    print(tag, rows, n3, "chunks", c.value, "chunk", ch.value, f"{dt*1e3:.2f} ms", flush=True)
np.savez(f"gpurun_out/ozaki_{tag}.npz", **{f"{k[0]}_{k[1]}": v for k, v in out.items()})
if tag == "ozaki" and os.path.exists("gpurun_out/ozaki_dmma.npz"):
    ref = np.load("gpurun_out/ozaki_dmma.npz")
    for k, v in out.items():
        r = ref[f"{k[0]}_{k[1]}"]
        d = np.abs(v - r).max() / np.abs(r).max()
        sym = np.abs(v - v.T).max()
        w1 = np.linalg.eigvalsh(r)[::-1][:8]
        w2 = np.linalg.eigvalsh(v)[::-1][:8]
        print("compare", k, "max|dG|/max|G|", d, "asym", sym, "eig rel", np.abs(w1 - w2).max() / w1[0])
