import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from golden_io import Case
import paper_1903_12294_b200 as P
import test_gpu_parity as T
for dbg in ("0", "1", "2", "3"):
    os.environ["MFSEG_DEBUG"] = dbg
    for name in ("assign_hard_2", "assign_hard_0", "assign_oracle_equiv"):
        case = Case(name)
        params = T._params(case); ext = T._extent(case)
        C = P.interval_distances(ext, params.k)
        cs = T._state(case, "in_c_")
        pl, fl = P.assign_iteration(T._points(case), T._field(case), None, cs, P.CenterGrid(cs.loc, ext, C, params.k), params, C)
        print("debug", dbg, name, "field mismatches", int((fl != case["out_field_labels"]).sum()))
