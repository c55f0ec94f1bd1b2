import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2409_19402_b200 as pp
from paper_2409_19402_b200 import synth, dist as pdist
a = synth.cp_tensor(96, 128, 64, rank=12, noise=1e-3, seed=11)
da = pp.to_device(a)
be = pdist.DeviceBackend("cuda:0")
plan = pdist.make_plan(96, 128, 64, 16, 1, 0, be)
print(plan)
Q, sig = be.sym_eig_top(be.tree_reduce(be.gram_partials(da, 96*128, 64, plan.chunk, plan.chunks_per_rank)), 64, 16)
Ah = be.mode3_fwd(da, 96, 128, 64, Q, 16)
U, s, V = be.svd_slices(Ah, 96, 128, 16, 6)
torch.cuda.synchronize()
print("s", s[:, :3].cpu())
f, re = pp.compress_tsvdq(da, 16, 6)
print("ref s", pp.to_host(f.s)[:, :3])
