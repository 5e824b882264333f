"""Per-pass phase times (grid, field, point, fallback, update; ms) of a run on the
bench's data, from runs stopped after 1, 2, ... passes (the runs are deterministic).
Usage: python tools/pass_times.py [config] [max_iterations]"""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS, rank_data, workload
from paper_1903_12294_b200 import ClusterParams, _native as N
from paper_1903_12294_b200.engine import run_device
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = CONFIGS[name]
fld, pts, _, _, _ = rank_data(cfg, 1, 0, 0, torch.device("cuda", 0))
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
lib = N.load()
prev = [0.0] * 5
for p in range(1, iters + 1):
    params = ClusterParams(k=workload(cfg, 1)[3], eps_c=1e-12, max_iterations=p)
    run_device(pts, fld, ext, params); torch.cuda.synchronize()
    best = None
    for _ in range(3):
        lib.mfseg_timing_enable(1)
        run_device(pts, fld, ext, params); torch.cuda.synchronize()
        ph = (C.c_double * 8)(); lib.mfseg_timing_read(ph, 8); lib.mfseg_timing_enable(0)
        cur = [ph[i] for i in range(5)]
        best = cur if best is None or sum(cur) < sum(best) else best
    print(f"pass {p}: " + " ".join(f"{b - a:7.3f}" for a, b in zip(prev, best)), flush=True)
    prev = best
