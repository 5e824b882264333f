import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from bench import CONFIGS, rank_data, workload
from paper_1903_12294_b200 import ClusterParams
from paper_1903_12294_b200.engine import run_device
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
from paper_1903_12294_b200.postproc import merge_device
cfg = CONFIGS["c2"]
fld, pts, tid, _, _ = rank_data(cfg, 1, 0, 0, torch.device("cuda", 0))
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
r = run_device(pts, fld, ext, ClusterParams(k=workload(cfg, 1)[3], eps_c=1e-12, max_iterations=10))
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); out = merge_device(r.state, 0.05); b.record(); torch.cuda.synchronize()
    print(f"merge_device events {a.elapsed_time(b):.2f} ms wall {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
