"""Random shapes through the star-Q host pipeline (2-D tiles): bitwise the
device call, and both within 1e-12 of a numpy FP64 product.

  python tools/starq_host_stress.py [cases] [seed]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_19402_b200 as pp  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for c in range(cases):
    n1 = int(rng.integers(1, 700))
    n2 = int(rng.integers(1, 700))
    m = int(rng.choice([64, 256, 320, 512]))
    n3 = int(rng.choice([32, 64, 96]))
    p = int(rng.choice([8, 16, 32, 64]))
    p = min(p, n3)
    a = np.asfortranarray(rng.standard_normal((n1, m, n3)))
    b = np.asfortranarray(rng.standard_normal((m, n2, n3)))
    kind = int(rng.integers(0, 4))
    if kind == 1 and n1 > 130:   # a row block of A with a huge dynamic range
        a[129, 3, :] *= 1e9
    if kind == 2:                # a late lateral block of B fails the gate
        b[5, n2 - 1, :] *= 1e9
    if kind == 3 and n2 > 2:     # an early one
        b[5, 1, :] *= 1e9
    t = pp.Transform("dct", n3, p)
    dev = pp.to_host(pp.star_q(pp.to_device(a), pp.to_device(b), t))
    host = pp.star_q(a, b, t)
    q = t.q
    ah = np.einsum("imk,kp->imp", a, q)
    bh = np.einsum("mjk,kp->mjp", b, q)
    want = np.einsum("ijp,kp->ijk", np.einsum("imp,mjp->ijp", ah, bh), q)
    err = np.linalg.norm(dev - want) / max(np.linalg.norm(want), 1e-300)
    same = np.array_equal(dev, host)
    flag = "" if (same and err <= 1e-12) else "   <-- FAIL"
    bad += bool(flag)
    print(f"case {c:2d} n1={n1:3d} m={m:3d} n2={n2:3d} n3={n3:2d} p={p:2d} kind={kind} bitwise={same} err={err:.1e}{flag}",
          flush=True)
print("failures:", bad)
sys.exit(1 if bad else 0)
