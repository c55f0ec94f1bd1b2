import sys; sys.path.insert(0,'.')
import paper_2409_19402_b200 as pp
from paper_2409_19402_b200 import synth
for shape,p,k,noise,rank in [((128,128,64),48,16,1e-2,20),((128,128,64),48,18,1e-2,20),((128,128,64),48,19,3e-2,20),((128,96,64),32,12,1e-2,16),((128,96,64),32,14,2e-2,16),((160,128,64),40,8,5e-2,10)]:
    a = synth.cp_tensor(*shape, rank=rank, noise=noise, seed=5)
    da = pp.to_device(a)
    f, re = pp.compress_tsvdq(da, p, k)
    print(shape,p,k,noise,rank, re, re*re)
