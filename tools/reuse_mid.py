import os, sys
sys.path.insert(0, "/root/repo")
os.environ["MFSEG_DEBUG"] = "8"
import paper_1903_12294_b200 as P
from paper_1903_12294_b200 import _native as _N; _N.debug_options_from_env()  # MFSEG_* knobs
from paper_1903_12294_b200.engine import run_device
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device, synthetic_device
fld, pts, _ = synthetic_device((128, 96, 64), 24, 20000, seed=5, noise=0.05, n_blobs=3, dyadic=False)
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
params = P.ClusterParams(k=(8, 6, 4, 6), eps_c=1e-12, max_iterations=10)
a = run_device(pts, fld, ext, params)
print("iters", a.iterations_used)
