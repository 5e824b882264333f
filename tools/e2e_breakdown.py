import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
import paper_1903_12294_b200 as P
from paper_1903_12294_b200.engine import points_to_device, field_to_device, run_device, CenterState, to_host
from paper_1903_12294_b200.ingest import synthetic_device, normalize_device, domain_extent_device
cfg = CONFIGS["c2"]
fld, pts, _ = synthetic_device(cfg["dims"], cfg["nt"], cfg["n_traj"], seed=0)
fv = torch.empty(fld.values.shape, dtype=torch.float64, pin_memory=True); fv.copy_(fld.values)
xyz = torch.empty(pts.xyz.shape, dtype=torch.float64, pin_memory=True); xyz.copy_(pts.xyz)
pt = torch.empty(pts.t.shape, dtype=torch.float64, pin_memory=True); pt.copy_(pts.t)
pv = torch.empty(pts.value.shape, dtype=torch.float64, pin_memory=True); pv.copy_(pts.value)
nt = cfg["nt"]
fields = P.FieldSet(tuple(cfg["dims"]), np.zeros(3), np.ones(3), np.arange(nt, dtype=float), fv.numpy().reshape(nt, -1))
points = P.PointSet(np.zeros(pts.n, np.int64), pt.numpy(), xyz.numpy(), pv.numpy())
print("pinned check:", torch.from_numpy(fv.numpy()).is_pinned(), flush=True)
params = P.ClusterParams(k=cfg["k"], eps_c=1e-12, max_iterations=10)
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = T(); d_p = points_to_device(points); d_f = field_to_device(fields); t1 = T()
    norm = normalize_device(d_p, d_f, True); t2 = T()
    ext = domain_extent_device(d_p, d_f); t3 = T()
    r = run_device(d_p, d_f, ext, params); t4 = T()
    st = CenterState.from_device(r.state); t5 = T()
    pl = to_host(r.point_labels); fl = to_host(r.field_labels); t6 = T()
    tab = st.to_table(); t7 = T()
    print(f"h2d {t1-t0:.3f} norm {t2-t1:.3f} extent {t3-t2:.3f} run {t4-t3:.3f} state {t5-t4:.3f} labels {t6-t5:.3f} table {t7-t6:.3f} total {t7-t0:.3f}", flush=True)
    del d_p, d_f, r
