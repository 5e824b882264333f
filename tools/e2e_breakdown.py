"""Where the public-API end-to-end time goes (segment() on pinned host arrays, c2)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
import paper_1903_12294_b200 as P
from paper_1903_12294_b200 import pipeline as PL
from paper_1903_12294_b200.engine import points_to_device, field_to_device, CenterState, to_host
from paper_1903_12294_b200.ingest import synthetic_device
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
fld, pts, _ = synthetic_device(cfg["dims"], cfg["nt"], cfg["n_traj"], seed=0)
pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)
fv, xyz, pt, pv = pin(fld.values), pin(pts.xyz), pin(pts.t), pin(pts.value)
nt = cfg["nt"]
fields = P.FieldSet(tuple(cfg["dims"]), np.zeros(3), np.ones(3), np.arange(nt, dtype=float), fv.numpy().reshape(nt, -1))
points = P.PointSet(np.zeros(pts.n, np.int64), pt.numpy(), xyz.numpy(), pv.numpy())
params = P.ClusterParams(k=cfg["k"], eps_c=1e-12, max_iterations=10)
del fld, pts
torch.cuda.empty_cache()
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(5):
    t0 = T(); d_p = points_to_device(points); d_f = field_to_device(fields); t1 = T()
    from paper_1903_12294_b200.ingest import normalize_device, domain_extent_device
    from paper_1903_12294_b200.engine import run_device
    from paper_1903_12294_b200.ingest import minmax_normalize_
    tq0 = T(); minmax_normalize_(d_p.value, "point"); tq1 = T(); minmax_normalize_(d_f.values, "field"); ta = T()
    print(f"  minmax point {tq1-tq0:.3f} field {ta-tq1:.3f}", flush=True)
    ext = domain_extent_device(d_p, d_f); tb = T()
    r = run_device(d_p, d_f, ext, params); t2 = T()
    ms = torch.cuda.memory_stats()
    print(f"  norm {ta-t1:.3f} extent {tb-ta:.3f} run {t2-tb:.3f} retries {ms['num_alloc_retries']} "
          f"device allocs {ms.get('num_device_alloc', -1)} frees {ms.get('num_device_free', -1)} "
          f"reserved {torch.cuda.memory_reserved()/1e9:.1f} GB", flush=True)
    st = CenterState.from_device(r.state); t3 = T()
    pl = to_host(r.point_labels); fl = to_host(r.field_labels); t4 = T()
    tab = st.to_table(); t5 = T()
    print(f"h2d {t1-t0:.3f} norm+extent+run {t2-t1:.3f} state {t3-t2:.3f} labels {t4-t3:.3f} "
          f"table {t5-t4:.3f} total {t5-t0:.3f}", flush=True)
    del d_p, d_f, r
for rep in range(3):
    t0 = T(); seg, _, _ = P.segment(points, fields, params); t1 = T()
    ms = torch.cuda.memory_stats()
    print(f"segment() {t1-t0:.3f} retries {ms['num_alloc_retries']} device allocs {ms.get('num_device_alloc', -1)} "
          f"frees {ms.get('num_device_free', -1)}", flush=True)
