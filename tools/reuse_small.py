import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
os.environ["MFSEG_DEBUG"] = "8"
import numpy as np
import paper_1903_12294_b200 as P
from paper_1903_12294_b200 import _native as _N; _N.debug_options_from_env()  # MFSEG_* knobs
from paper_1903_12294_b200.ingest import synthetic_device
dims, nt, ntraj = (64, 48, 40), 8, 2000
fld, pts, _ = synthetic_device(dims, nt, ntraj, seed=31, noise=0.05, n_blobs=5, dyadic=False)
fs = P.FieldSet(dims, np.zeros(3), np.ones(3), fld.times.cpu().numpy(), fld.values.cpu().numpy().reshape(nt, -1))
ps = P.PointSet(np.zeros(pts.n, np.int64), pts.t.cpu().numpy(), pts.xyz.cpu().numpy(), pts.value.cpu().numpy())
ext = P.domain_extent(ps, fs)
params = P.ClusterParams(k=(5, 4, 3, 2), w_d=0.3, max_iterations=5, eps_c=1e-12)
a = P.run(ps, fs, ext, params)
