"""Micro-timings of the e2e pieces that showed spikes (normalize, to_host)."""
import os, sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
from paper_1903_12294_b200.engine import to_host
from paper_1903_12294_b200.ingest import synthetic_device, minmax_normalize_
cfg = CONFIGS["c2"]
fld, pts, _ = synthetic_device(cfg["dims"], cfg["nt"], cfg["n_traj"], seed=0)
def T(): torch.cuda.synchronize(); return time.perf_counter()
print("gc thresholds", gc.get_threshold(), flush=True)
for i in range(8):
    t0 = T(); minmax_normalize_(fld.values, "field", apply=False); t1 = T()
    minmax_normalize_(pts.value, "point", apply=False); t2 = T()
    print(f"minmax field {t1-t0:.4f} point {t2-t1:.4f}", flush=True)
lab = torch.zeros(fld.values.numel(), dtype=torch.int32, device="cuda")
keep = []
for i in range(6):
    t0 = T(); h = to_host(lab); t1 = T()
    keep.append(h)
    if len(keep) > 2: keep.pop(0)
    print(f"to_host 2.1GB {t1-t0:.4f}", flush=True)
