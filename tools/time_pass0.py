"""Initial-pass cost with and without the interior shortcut (debug flag
NO_SEEDS_FAST), bench data on one GPU.  Usage: python tools/time_pass0.py [config]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS, rank_data, workload
from paper_1903_12294_b200 import ClusterParams
from paper_1903_12294_b200 import _native as N
from paper_1903_12294_b200.engine import run_device
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
fld, pts, _, _, _ = rank_data(cfg, 1, 0, 0, torch.device("cuda", 0))
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
for iters in (1, 2):
    params = ClusterParams(k=workload(cfg, 1)[3], eps_c=1e-12, max_iterations=iters)
    res = {}
    for name, flags in (("fast", 0), ("full", N.DEBUG_NO_SEEDS_FAST)):
        ts = []
        with N.debug_options(flags):
            for _ in range(4):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                r = run_device(pts, fld, ext, params)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
        res[name] = r
        print(f"iters={iters} {name}: " + " ".join(f"{t:.2f}" for t in ts) + " ms", flush=True)
    a, b = res["fast"], res["full"]
    print("  labels equal:", torch.equal(a.field_labels, b.field_labels), torch.equal(a.point_labels, b.point_labels))
