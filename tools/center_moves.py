"""Per-pass centre movement on bench data: max |delta loc| per axis in units of
the bin size C, and the max relative change reported by the engine.
Usage: python tools/center_moves.py [config] [iterations]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
from paper_1903_12294_b200 import ClusterParams, interval_distances
from paper_1903_12294_b200.engine import run_device, CenterState
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device, synthetic_device
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
fld, pts, _ = synthetic_device(cfg["dims"], cfg["nt"], cfg["n_traj"], seed=0)
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
C = np.array(interval_distances(ext, cfg["k"]))
prev = None
for it in range(1, iters + 1):
    params = ClusterParams(k=cfg["k"], eps_c=1e-12, max_iterations=it)
    r = run_device(pts, fld, ext, params)
    st = CenterState.from_device(r.state)
    loc = np.asarray(st.loc)
    fv = np.asarray(st.fval)
    if prev is not None:
        d = np.abs(loc - prev[0]) / C
        dv = np.nanmax(np.abs(fv - prev[1]))
        q = np.quantile(d.max(axis=1), [0.5, 0.9, 0.99, 1.0])
        print(f"pass {it}: |dloc|/C per-centre max: median {q[0]:.2e} p90 {q[1]:.2e} p99 {q[2]:.2e} max {q[3]:.2e}; max |dfval| {dv:.2e}", flush=True)
        # sample bins whose 3^4 neighbourhood holds no centre that changed
        k = np.array(cfg["k"])
        mins = np.array([ext.xmin, ext.ymin, ext.zmin, ext.tmin])
        moved = (np.abs(loc - prev[0]).max(axis=1) > 0) | ~((fv == prev[1]) | (np.isnan(fv) & np.isnan(prev[1])))
        b = np.clip(np.floor((loc - mins) / C), 0, k - 1).astype(int)
        grid = np.zeros(k[::-1], bool)   # [t, z, y, x]
        np.logical_or.at(grid, (b[moved, 3], b[moved, 2], b[moved, 1], b[moved, 0]), True)
        pad = np.pad(grid, 1)
        nb = np.zeros_like(grid)
        for dt in range(3):
            for dz in range(3):
                for dy in range(3):
                    for dx in range(3):
                        nb |= pad[dt:dt + k[3], dz:dz + k[2], dy:dy + k[1], dx:dx + k[0]]
        print(f"   moved centres {moved.mean():.3f}; bins with an unchanged 3^4 neighbourhood {1 - nb.mean():.3f}", flush=True)
    prev = (loc, fv)

