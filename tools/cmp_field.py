"""Full run of a config with field kernels v1 / v4 / v5: labels must be identical,
centres equal to rounding (value sums are fixed-order fp64 per warp).
Usage: python tools/cmp_field.py [config] [iterations] [versions...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
from paper_1903_12294_b200 import ClusterParams, _native as N
from paper_1903_12294_b200.engine import run_device, CenterState
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device, synthetic_device
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
vers = sys.argv[3:] or ["v4", "v5"]   # v1/v3/v4/v5 (field) or any MFSEG_* env name, "default"
fld, pts, _ = synthetic_device(cfg["dims"], cfg["nt"], cfg["n_traj"], seed=0)
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
params = ClusterParams(k=cfg["k"], eps_c=1e-12, max_iterations=iters)
lib = N.load()
res = {}
for tag in vers:
    for e in [x for x in os.environ if x.startswith("MFSEG_")]:
        os.environ.pop(e, None)
    if tag.startswith("MFSEG_"):
        os.environ[tag] = "1"
    elif tag not in ("v5", "default"):
        os.environ["MFSEG_FIELD_" + tag.upper()] = "1"
    r = run_device(pts, fld, ext, params)
    torch.cuda.synchronize()
    lib.mfseg_timing_enable(1)
    t0 = time.perf_counter(); r = run_device(pts, fld, ext, params); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    import ctypes as C
    ph = (C.c_double * 8)()
    lib.mfseg_timing_read(ph, 8)
    lib.mfseg_timing_enable(0)
    passes = r.iterations_used + 1
    res[tag] = (r.field_labels.clone(), r.point_labels.clone(), CenterState.from_device(r.state), dt)
    print(tag, "run %.3f s" % dt, "iters", r.iterations_used,
          "phase ms/pass", [round(ph[i] / passes, 3) for i in range(5)], flush=True)
base = vers[0]
for tag in vers[1:]:
    a, b = res[base], res[tag]
    print(base, "vs", tag, "field labels identical:", torch.equal(a[0], b[0]),
          "mismatches:", int((a[0] != b[0]).sum()), "point labels identical:", torch.equal(a[1], b[1]),
          "centres max rel diff:",
          float(np.nanmax(np.abs(a[2].loc - b[2].loc) / np.maximum(np.abs(a[2].loc), 1e-300))),
          "fval max abs diff:", float(np.nanmax(np.abs(a[2].fval - b[2].fval))), flush=True)
