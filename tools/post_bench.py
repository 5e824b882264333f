"""Post-processing timings at a bench config: merge_clusters + build_features
(relabel, GPU trajectory split, voxel CSR, feature stats) on a finished run."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS
import paper_1903_12294_b200 as P
from paper_1903_12294_b200.postproc import split_trajectories_device
from paper_1903_12294_b200.ingest import synthetic_device
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
fld, pts, tid = synthetic_device(cfg["dims"], cfg["nt"], cfg["n_traj"], seed=0)
nt = cfg["nt"]
fields = P.FieldSet(tuple(cfg["dims"]), np.zeros(3), np.ones(3), np.arange(nt, dtype=float),
                    fld.values.cpu().numpy().reshape(nt, -1))
points = P.PointSet(tid.cpu().numpy(), pts.t.cpu().numpy(), pts.xyz.cpu().numpy(), pts.value.cpu().numpy())
params = P.ClusterParams(k=cfg["k"], eps_c=1e-12, max_iterations=10)
def T(): torch.cuda.synchronize(); return time.perf_counter()
seg, norm, _ = P.segment(points, fields, params)
for rep in range(2):
    t0 = T(); mm, merged = P.merge_clusters(seg.centers, 0.05); t1 = T()
    slot = torch.as_tensor(seg.point_labels).cuda()
    t2 = T(); order, starts, stride = split_trajectories_device(tid, pts.t, slot); t3 = T()
    feats = P.build_features(seg, mm, points, fields); t4 = T()
    print(f"K={len(seg.centers)} merged={len(merged)} features={len(feats)} runs={starts.numel() - 1} | "
          f"merge {t1 - t0:.3f} s, traj_split (device) {1e3 * (t3 - t2):.1f} ms, "
          f"build_features (incl. host lists) {t4 - t3:.2f} s", flush=True)
if len(sys.argv) > 2 and sys.argv[2] == "profile":
    import cProfile, pstats
    cProfile.run("P.build_features(seg, mm, points, fields)", "/tmp/bf.prof")
    pstats.Stats("/tmp/bf.prof").sort_stats("cumulative").print_stats(18)
