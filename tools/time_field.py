"""Per-pass phase times of a full run under the current env (field kernel variants)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS
from paper_1903_12294_b200 import ClusterParams, _native as N
from paper_1903_12294_b200 import _native as _N; _N.debug_options_from_env()  # MFSEG_* knobs
from paper_1903_12294_b200.engine import run_device
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device, synthetic_device
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
from bench import rank_data, workload
fld, pts, _, _, _ = rank_data(cfg, 1, 0, 0, torch.device("cuda", 0))   # the bench's data
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
params = ClusterParams(k=workload(cfg, 1)[3], eps_c=1e-12, max_iterations=10)
lib = N.load()
for env in sys.argv[2:] or [""]:
    for e in [x for x in os.environ if x.startswith("MFSEG_")]:
        os.environ.pop(e)
    if env:
        os.environ[env] = "1"
    _N.debug_options_from_env()
    run_device(pts, fld, ext, params); torch.cuda.synchronize()
    lib.mfseg_timing_enable(1)
    r = run_device(pts, fld, ext, params); torch.cuda.synchronize()
    ph = (C.c_double * 8)(); lib.mfseg_timing_read(ph, 8); lib.mfseg_timing_enable(0)
    n = r.iterations_used + 1
    print(env or "default", "phase ms/pass", [round(ph[i] / n, 3) for i in range(5)], flush=True)
