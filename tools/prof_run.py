"""Profiling driver: bench data (bench.rank_data, one GPU), a short run
(initial pass + 2 weighted passes by default).
Usage: python tools/prof_run.py [config] [iterations]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS, rank_data, workload
from paper_1903_12294_b200 import ClusterParams
from paper_1903_12294_b200 import _native as _N; _N.debug_options_from_env()  # MFSEG_* knobs
from paper_1903_12294_b200.engine import run_device
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device, synthetic_device
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
fld, pts, _, _, _ = rank_data(cfg, 1, 0, 0, torch.device("cuda", 0))
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
params = ClusterParams(k=workload(cfg, 1)[3], eps_c=1e-12, max_iterations=iters)
r = run_device(pts, fld, ext, params)
torch.cuda.synchronize()
print("ok", r.iterations_used)
