import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2403_01778_b200 as r1
from oracle import rank1_oracle as O
dims=(100,100,100)
a=O.gen_config(1,dims,1)
o=r1.SolveOptions(tol=1e-300,max_iters=30,init="provided",init_factors=[np.ones(100)]*3,record_kkt=False)
rep=r1.solve("hoscf", r1.DenseTensor(dims,a), o)
print("iters", rep.iterations, rep.wall_eig())
