"""Generates tests/golden/cfg5_dmma.json (run once on a B200; ~10 min):
the BASELINE cfg5 tensor (2048x2048x1024 rank-50 CP + N(0,1e-3^2), seed 0,
synth.cp_tensor_device), its data-driven basis Q (p=128) from the engine's
all-FP64-DMMA path (ppc_set_ozaki(0)), and an independent relative error of
the rank-32 tSVDQ with that Q: A x3 Q^T is formed on the host (numpy BLAS)
and every one of its 128 slices is decomposed by LAPACK (numpy.linalg.svd),
RE^2 = (||A||^2 - ||Ahat||^2 + sum_i sum_{j>=k} s_ij^2) / ||A||^2
(Q orthonormal: decompositions.cpp:30-58 / metrics.cpp:21-28 restated).

  python tools/golden_cfg5.py tests/golden/cfg5_dmma.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19402_b200 as pp  # noqa: E402
from paper_2409_19402_b200 import synth  # noqa: E402


def main(out):
    n1, n2, n3, p, k = 2048, 2048, 1024, 128, 32
    A = synth.cp_tensor_device(n1, n2, n3, rank=50, noise=1e-3, seed=0)
    pp.set_fp64_only(True)
    f, re = pp.compress_tsvdq(A, p, k)
    pp.set_fp64_only(False)
    q = np.ascontiguousarray(f.transform.q)
    t0 = time.time()
    Ah = np.zeros((n1 * n2, p))
    a2 = 0.0
    for c0 in range(0, n3, 64):
        blk = A[:, :, c0:c0 + 64].permute(2, 1, 0).reshape(-1, n1 * n2).cpu().numpy()
        Ah += blk.T @ q[c0:c0 + 64]
        a2 += float(np.sum(blk * blk))
    lam = np.sum(Ah * Ah, axis=0)
    tail = 0.0
    for i in range(p):
        s = np.linalg.svd(Ah[:, i].reshape(n1, n2, order="F"), compute_uv=False)
        tail += float(np.sum(s[k:] ** 2))
    re_l = ((a2 - float(np.sum(lam))) + tail) ** 0.5 / a2 ** 0.5
    res = {"config": "cfg5 2048x2048x1024 rank-50 CP + N(0,1e-3^2), seed 0; p=128, k=32",
           "relative_error_engine_fp64": re, "relative_error_lapack": re_l,
           "lambda": [float(x) for x in lam], "host_seconds": time.time() - t0}
    with open(out, "w") as fo:
        json.dump(res, fo, indent=1)
    print(json.dumps({kk: v for kk, v in res.items() if kk != "lambda"}))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "tests/golden/cfg5_dmma.json")
