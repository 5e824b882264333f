"""Full c2 (or given config) run with the v1 and v2 field kernels: labels and centres must be identical."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
from paper_1903_12294_b200 import ClusterParams
from paper_1903_12294_b200.engine import run_device, CenterState
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device, synthetic_device
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
fld, pts, _ = synthetic_device(cfg["dims"], cfg["nt"], cfg["n_traj"], seed=0)
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
params = ClusterParams(k=cfg["k"], eps_c=1e-12, max_iterations=iters)
res = {}
for tag in ("v1", "v2", "v3"):
    for e in ("MFSEG_FIELD_V1", "MFSEG_POINT_V1", "MFSEG_FIELD_V3"):
        os.environ.pop(e, None)
    if tag == "v1":
        os.environ["MFSEG_FIELD_V1"] = "1"; os.environ["MFSEG_POINT_V1"] = "1"
    elif tag == "v2":
        os.environ["MFSEG_FIELD_V3"] = "1"
    r = run_device(pts, fld, ext, params)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); r = run_device(pts, fld, ext, params); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res[tag] = (r.field_labels.clone(), r.point_labels.clone(), CenterState.from_device(r.state), dt, r.iterations_used)
    print(tag, "run %.3f s" % dt, "iters", r.iterations_used, flush=True)
a, b = res["v1"], res["v3"]
print("field labels identical:", torch.equal(a[0], b[0]), "mismatches:", int((a[0] != b[0]).sum()))
print("point labels identical:", torch.equal(a[1], b[1]))
print("centres identical:", np.array_equal(a[2].loc, b[2].loc), "max rel diff:",
      float(np.nanmax(np.abs(a[2].loc - b[2].loc) / np.maximum(np.abs(a[2].loc), 1e-300))))
