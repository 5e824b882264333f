import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from golden_io import Case
import paper_1903_12294_b200 as P
import test_gpu_parity as T
os.environ["MFSEG_DEBUG"] = "4"
case = Case("assign_hard_2")
params = T._params(case); ext = T._extent(case)
C = P.interval_distances(ext, params.k)
cs = T._state(case, "in_c_")
print("centres x:", cs.loc[:, 0])
pl, fl = P.assign_iteration(T._points(case), T._field(case), None, cs, P.CenterGrid(cs.loc, ext, C, params.k), params, C)
import torch; torch.cuda.synchronize()
