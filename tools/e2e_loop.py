"""segment() called repeatedly like bench's e2e: per-call time and host-allocator stats."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
import paper_1903_12294_b200 as P
from paper_1903_12294_b200.ingest import synthetic_device
cfg = CONFIGS["c2"]
fld, pts, _ = synthetic_device(cfg["dims"], cfg["nt"], cfg["n_traj"], seed=0)
pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)
fv, xyz, pt, pv = pin(fld.values), pin(pts.xyz), pin(pts.t), pin(pts.value)
nt = cfg["nt"]
fields = P.FieldSet(tuple(cfg["dims"]), np.zeros(3), np.ones(3), np.arange(nt, dtype=float), fv.numpy().reshape(nt, -1))
points = P.PointSet(np.zeros(pts.n, np.int64), pt.numpy(), xyz.numpy(), pv.numpy())
params = P.ClusterParams(k=cfg["k"], eps_c=1e-12, max_iterations=10)
del fld, pts
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    seg, _, _ = P.segment(points, fields, params)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    try:
        hs = torch.cuda.host_memory_stats()
        extra = f"host allocs {hs.get('num_host_alloc', '?')} frees {hs.get('num_host_free', '?')} " \
                f"alloc_time {hs.get('host_alloc_time.total', '?')}"
    except Exception as e:
        extra = str(e)[:60]
    print(f"call {i}: {dt:.3f} s  {extra}", flush=True)

# --- the bench's order: device-resident runs first, then e2e calls with a stage breakdown
if len(sys.argv) > 1:
    from paper_1903_12294_b200 import pipeline as PL
    from paper_1903_12294_b200.engine import points_to_device, field_to_device
    orig = PL.segment_device
    def timed_segment_device(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = orig(*a, **k)
        torch.cuda.synchronize(); print(f"   segment_device {time.perf_counter() - t0:.3f}", flush=True)
        return r
    PL.segment_device = timed_segment_device
    orig_ts = PL.to_segmentation
    def timed_ts(*a, **k):
        t0 = time.perf_counter(); r = orig_ts(*a, **k); print(f"   to_segmentation {time.perf_counter() - t0:.3f}", flush=True); return r
    PL.to_segmentation = timed_ts
    for i in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        seg, _, _ = P.segment(points, fields, params)
        torch.cuda.synchronize(); print(f"call {i}: {time.perf_counter() - t0:.3f} s", flush=True)

if len(sys.argv) > 2:
    from paper_1903_12294_b200.ingest import normalize_device, domain_extent_device
    from paper_1903_12294_b200.engine import run_device, points_to_device, field_to_device
    def T(): torch.cuda.synchronize(); return time.perf_counter()
    for i in range(10):
        t0 = T(); dp = points_to_device(points); df = field_to_device(fields); t1 = T()
        normalize_device(dp, df, True); t2 = T()
        ext = domain_extent_device(dp, df); t3 = T()
        r = run_device(dp, df, ext, params); t4 = T()
        ms = torch.cuda.memory_stats()
        print(f"iter {i}: h2d {t1-t0:.3f} norm {t2-t1:.3f} ext {t3-t2:.3f} run {t4-t3:.3f} "
              f"allocs {ms.get('num_device_alloc')} frees {ms.get('num_device_free')} retries {ms['num_alloc_retries']}", flush=True)
        del dp, df, r
