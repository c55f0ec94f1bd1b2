import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PPC_SUBSPACE_DEBUG"] = "1"
import paper_2409_19402_b200 as pp
from paper_2409_19402_b200 import synth
from oracle import ppo
a = synth.video(240, 320, 40, seed=4)
q, _, _ = ppo.data_dependent_q(a, 12)
ah = np.asfortranarray(np.einsum("ijk,kl->ijl", a, q))
for k in (1, 20):
    U, s, V = pp.truncated_svd(ah, k)
    for z in range(12):
        sn = np.linalg.svd(ah[:, :, z], compute_uv=False)[:k]
        print("k", k, "slice", z, "max rel sigma err", np.max(np.abs(s[:, z] - sn) / sn))
