"""Whole-run CUDA-event time against the sum of the per-pass phase times (the rest is the
one-off preparation plus host gaps between passes).  Usage: python tools/run_gaps.py c2"""
import os, sys, ctypes as C
sys.path.insert(0, "/root/repo")
import torch
from bench import CONFIGS, rank_data, workload
from paper_1903_12294_b200 import ClusterParams, _native as N
from paper_1903_12294_b200.engine import run_device
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
cfg = CONFIGS[sys.argv[1]]
fld, pts, _, _, _ = rank_data(cfg, 1, 0, 0, torch.device("cuda", 0))
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
lib = N.load()
for iters in (1, 2, 10):
    params = ClusterParams(k=workload(cfg, 1)[3], eps_c=1e-12, max_iterations=iters)
    run_device(pts, fld, ext, params); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = run_device(pts, fld, ext, params); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    lib.mfseg_timing_enable(1)
    r = run_device(pts, fld, ext, params); torch.cuda.synchronize()
    ph = (C.c_double * 8)(); lib.mfseg_timing_read(ph, 8); lib.mfseg_timing_enable(0)
    print(iters, "run ms", [round(t, 3) for t in ts], "phase sum", round(sum(ph[i] for i in range(5)), 3), [round(ph[i], 3) for i in range(5)], "passes", r.iterations_used + 1, flush=True)
