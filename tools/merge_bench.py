"""Timing of the device merge (mfseg_merge via postproc.merge_device) on the final
centres of a bench run, repeated (the union-find's atomics make it noisy).
Usage: python tools/merge_bench.py [config] [eps_m]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS, rank_data, workload
from paper_1903_12294_b200 import ClusterParams
from paper_1903_12294_b200.engine import run_device
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
from paper_1903_12294_b200.postproc import merge_device
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
fld, pts, _, _, _ = rank_data(cfg, 1, 0, 0, torch.device("cuda", 0))
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
r = run_device(pts, fld, ext, ClusterParams(k=workload(cfg, 1)[3], eps_c=1e-12, max_iterations=10))
ts = []
for _ in range(7):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ids, rep, merged = merge_device(r.state, eps)
    torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0))
print(f"merge of {ids.numel()} live centres -> {merged['ids'].numel()} features: "
      f"ms {[round(t, 2) for t in ts]}, median {sorted(ts)[3]:.2f}")
