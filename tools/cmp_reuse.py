"""A full run with and without reuse of stable field blocks (MFSEG_NO_REUSE):
labels and centres must be bit-identical.  Usage: python tools/cmp_reuse.py [config] [iterations]"""
import os, sys, subprocess, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 3:   # child: one run, save outputs
    import numpy as np, torch
    from bench import CONFIGS
    from paper_1903_12294_b200 import ClusterParams
    from paper_1903_12294_b200 import _native as _N; _N.debug_options_from_env()  # MFSEG_* knobs
    from paper_1903_12294_b200.engine import run_device, CenterState
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device, synthetic_device
    cfg = CONFIGS[sys.argv[1]]
    fld, pts, _ = synthetic_device(cfg["dims"], cfg["nt"], cfg["n_traj"], seed=0)
    normalize_device(pts, fld, True)
    ext = domain_extent_device(pts, fld)
    extra = {}
    for kv in filter(None, os.environ.get("CMP_WEIGHTS", "").split(",")):   # e.g. c_f=0.5,w_f=2
        key, val = kv.split("=")
        extra[key] = float(val)
    params = ClusterParams(k=cfg["k"], eps_c=1e-12, max_iterations=int(sys.argv[2]), **extra)
    r = run_device(pts, fld, ext, params)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = run_device(pts, fld, ext, params)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = CenterState.from_device(r.state)
    np.savez(sys.argv[3], fl=r.field_labels.cpu().numpy(), pl=r.point_labels.cpu().numpy(),
             loc=np.asarray(st.loc), fv=np.asarray(st.fval), pv=np.asarray(st.pval))
    print(f"{os.environ.get('MFSEG_NO_REUSE', 'reuse')}: run {dt*1e3:.1f} ms")
    sys.exit(0)
import numpy as np
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = sys.argv[2] if len(sys.argv) > 2 else "10"
env = dict(os.environ)
subprocess.run([sys.executable, __file__, cfgname, iters, "/tmp/reuse_a.npz"], env=env, check=True)
env["MFSEG_NO_REUSE"] = "1"
subprocess.run([sys.executable, __file__, cfgname, iters, "/tmp/reuse_b.npz"], env=env, check=True)
a, b = np.load("/tmp/reuse_a.npz"), np.load("/tmp/reuse_b.npz")
for k in a.files:
    same = np.array_equal(a[k], b[k], equal_nan=True) if a[k].dtype.kind == "f" else np.array_equal(a[k], b[k])
    print(k, "identical" if same else "DIFFERENT")
