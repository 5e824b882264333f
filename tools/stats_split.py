import sys, os, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from bench import CONFIGS, rank_data, workload
from paper_1903_12294_b200 import ClusterParams
from paper_1903_12294_b200.engine import run_device
from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
from paper_1903_12294_b200.postproc import feature_slots_device, feature_stats_device, merge_device
cfg = CONFIGS["c2"]
fld, pts, tid, _, _ = rank_data(cfg, 1, 0, 0, torch.device("cuda", 0))
normalize_device(pts, fld, True)
ext = domain_extent_device(pts, fld)
params = ClusterParams(k=workload(cfg, 1)[3], eps_c=1e-12, max_iterations=10)
r = run_device(pts, fld, ext, params)
ids, rep, merged = merge_device(r.state, 0.05)
fids = torch.unique(rep)
K = int(r.state["pval"].numel())
lut = np.full(K, -1, np.int64)
lut[ids.cpu().numpy()] = torch.searchsorted(fids, rep).cpu().numpy()
fslot = feature_slots_device(r.field_labels, lut)
pslot = feature_slots_device(r.point_labels, lut)
ns = int(fids.numel())
from paper_1903_12294_b200.engine import DevicePoints, DeviceField
def T(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); return 1e3 * (time.perf_counter() - t0)
z = torch.zeros(0, dtype=torch.float64, device="cuda")
nop = DevicePoints(z.reshape(0, 3), z, z)
nof = DeviceField(fld.dims, fld.origin, fld.spacing, z, z)
for _ in range(2):
    a = T(lambda: feature_stats_device(ns, fld, fslot, nop, None))
    b = T(lambda: feature_stats_device(ns, nof, None, pts, pslot))
    order = torch.argsort(pslot, stable=True)
    sp = DevicePoints(pts.xyz[order].contiguous(), pts.t[order].contiguous(), pts.value[order].contiguous())
    c = T(lambda: feature_stats_device(ns, nof, None, sp, pslot[order].contiguous()))
    d = T(lambda: torch.argsort(pslot, stable=True))
print(f"fields only {a:.2f} ms, points only {b:.2f} ms, points sorted by slot {c:.2f} ms, argsort {d:.2f} ms")
