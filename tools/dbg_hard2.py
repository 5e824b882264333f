import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from golden_io import Case
import paper_1903_12294_b200 as P
import test_gpu_parity as T
from oracle import mfseg_oracle as O
case = Case("assign_hard_2")
params = T._params(case); ext = T._extent(case)
C = P.interval_distances(ext, params.k)
cs = T._state(case, "in_c_")
pl, fl = P.assign_iteration(T._points(case), T._field(case), None, cs, P.CenterGrid(cs.loc, ext, C, params.k), params, C)
exp = case["out_field_labels"]
dims, origin, spacing, times, values = case.field
floc = O.field_locations(dims, origin, spacing, times)
v = values.reshape(-1)
print("params", case.meta["params"], "dims", dims, "nt", len(times))
bad = np.flatnonzero(fl != exp)
for s in bad[:12]:
    D = O.distance_matrix(floc[s:s+1], v[s:s+1], cs.loc, cs.fval, cs.has_f, params.w_f, params.w_d, params.c_f)[0]
    inbox = np.all(np.abs(cs.loc - floc[s]) <= C, axis=1)
    tb = O.NeighbourTable(cs.loc, ext.mins, C, params.k)
    cand = tb.candidates(O.bins_of(floc[s:s+1], ext.mins, C, params.k)[0])
    print(s, "loc", floc[s], "got", fl[s], "exp", exp[s], "D_got %.17g D_exp %.17g" % (D[fl[s]], D[exp[s]]),
          "inbox got", inbox[fl[s]], "exp", inbox[exp[s]], "cand got", fl[s] in cand, "exp", exp[s] in cand)
