"""cfg2 video slice SVDs (k=20) with PPC_SUBSPACE_DEBUG=1 (stderr)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PPC_SUBSPACE_DEBUG", "1")
import torch  # noqa: E402
import paper_2409_19402_b200 as pp  # noqa: E402
from paper_2409_19402_b200 import synth  # noqa: E402

a = pp.to_device(synth.video(240, 320, 200, seed=0))
t = pp.data_dependent_transform(a, 20)
for k in (20, 10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = pp.tsvdq(a, t, k)
    torch.cuda.synchronize()
    print("k", k, "ms", (time.perf_counter() - t0) * 1e3)
