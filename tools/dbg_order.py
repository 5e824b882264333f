import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from golden_io import Case, names
import paper_1903_12294_b200 as P
import test_gpu_parity as T
for name in names("assign_"):
    case = Case(name)
    params = T._params(case); ext = T._extent(case)
    C = P.interval_distances(ext, params.k)
    cs = T._state(case, "in_c_")
    pl, fl = P.assign_iteration(T._points(case), T._field(case), None, cs, P.CenterGrid(cs.loc, ext, C, params.k), params, C)
    print(name, np.array_equal(pl, case["out_point_labels"]), np.array_equal(fl, case["out_field_labels"]),
          pl[:5], case["out_point_labels"][:5])
