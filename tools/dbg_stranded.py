import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_1903_12294_b200 as P
ext = P.DomainExtent(0, 16, 0, 1, 0, 1, 0, 1)
params = P.ClusterParams(k=(8, 1, 1, 1), w_d=1.0, w_p=1.0)
cs = P.CenterState.from_seeds(np.array([[1.0, 0.5, 0.5, 0.5], [3.0, 0.5, 0.5, 0.5]]))
cs.pval = np.array([0.9, 0.1]); cs.has_p = np.array([True, True])
C = P.interval_distances(ext, params.k)
for xs in ([15.0], [15.0, 14.0], [2.0, 15.0]):
    loc = np.array([[x, 0.5, 0.5, 0.5] for x in xs])
    pts = P.PointSet(np.arange(len(xs)), loc[:, 3].copy(), loc[:, :3].copy(), np.full(len(xs), 0.1))
    pl, fl = P.assign_iteration(pts, P.FieldSet.empty(), None, cs, P.CenterGrid(cs.loc, ext, C, params.k), params, C)
    print(xs, pl)
