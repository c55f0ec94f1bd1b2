"""Repeated host-buffer calls (star-Q pipeline, compress, sweep): device memory
in use and the host RSS must not grow (run on a B200: python tools/leak_check.py)."""
import os, sys, resource
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_2409_19402_b200 as pp
rng = np.random.default_rng(0)
a = np.asfortranarray(rng.standard_normal((300, 256, 32)))
b = np.asfortranarray(rng.standard_normal((256, 450, 32)))
t = pp.Transform("dct", 32, 16)
x = np.asfortranarray(rng.standard_normal((96, 80, 48)))
def snap():
    free, total = torch.cuda.mem_get_info()
    return (total - free) / 2**20, resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024
for i in range(5):
    pp.star_q(a, b, t); pp.compress_tsvdq(x, 12, 5)
torch.cuda.synchronize()
d0, h0 = snap()
for i in range(300):
    pp.star_q(a, b, t)
    pp.compress_tsvdq(x, 12, 5)
    pp.tsvdq_sweep(x, [12], [1, 3, 5])
torch.cuda.synchronize()
d1, h1 = snap()
print(f"device MiB used {d0:.0f} -> {d1:.0f}; host max RSS MiB {h0:.0f} -> {h1:.0f}")
assert d1 - d0 < 64 and h1 - h0 < 256, "leak?"
print("ok")
