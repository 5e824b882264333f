"""Multi-rank segmentation and feature materialisation on the GPU path.

Two ranks run as two processes on cuda:0 with the gloo backend: the per-pass
exchange and the post-processing collectives are host-side (gloo), and no
kernel waits on another rank's kernel, so sharing one GPU is safe.  For time
slabs (configs[2]) and spatial z-slabs (configs[4]), with and without
normalisation: labels, centres, the NormalizationRecord and every feature
(statistics, voxels, polylines, isolated points) must equal the single-GPU
`segment` + `build_features` bit for bit.  A one-rank NCCL group covers each
split through the NCCL backend.
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _dataset(seed=11, dims=(24, 20, 32), nt=12, ntraj=400):
    import paper_1903_12294_b200 as P
    from paper_1903_12294_b200.ingest import synthetic_device
    fld, pts, tid = synthetic_device(dims, nt, ntraj, seed=seed, noise=0.05, n_blobs=4)
    fs = P.FieldSet(dims, np.zeros(3), np.ones(3), np.arange(nt, dtype=float),
                    fld.values.cpu().numpy().reshape(nt, -1))
    ps = P.PointSet(tid.cpu().numpy(), pts.t.cpu().numpy(), pts.xyz.cpu().numpy(),
                    pts.value.cpu().numpy())
    return ps, fs


K_GRID = (3, 3, 4, 4)


def _params(normalize):
    import paper_1903_12294_b200 as P
    return P.ClusterParams(k=K_GRID, w_d=0.7, eps_c=1e-12, max_iterations=6, normalize=normalize)


def _features_digest(feats):
    out = {}
    for f in feats:
        out[f.id] = {"members": list(f.member_clusters),
                     "stats": f.stats.to_dict(),
                     "voxels": {int(m): np.asarray(c).tolist() for m, c in f.voxels.items()},
                     "polylines": [np.asarray(p).tolist() for p in f.polylines],
                     "isolated": [int(i) for i in f.isolated_points]}
    return out


def _rank_fn(rank, world, port, axis, normalize, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1903_12294_b200 as P
        from paper_1903_12294_b200.parallel import segment_sharded, shard_dataset
        from paper_1903_12294_b200.postproc import build_features_sharded
        ps, fs = _dataset()
        params = _params(normalize)
        lps, lfs, off, gd, idx, m0 = shard_dataset(ps, fs, params.k, rank, world, axis)
        seg, norm, _ = segment_sharded(lps, lfs, params, field_offset=off, grid_dims=gd)
        mm, _ = P.merge_clusters(seg.centers, 0.05)
        feats = build_features_sharded(seg, mm, lps, lfs, point_index=idx, field_offset=off,
                                       timestep_offset=m0, grid_dims=gd)
        q.put((rank, dict(fl=seg.field_labels, pl=seg.point_labels, idx=idx, off=off,
                          nz=lfs.dims[2], centers=[c.__dict__ for c in seg.centers],
                          norm=norm.to_dict(), it=seg.iterations_used,
                          feats=_features_digest(feats))))
    except BaseException as e:   # surfaced by the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(world, axis, normalize):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_fn, args=(r, world, port, axis, normalize, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert "error" not in out[r], out[r]["error"]
    return [out[r] for r in range(world)]


def _merge_digests(parts):
    """Rank-order concatenation of the per-rank feature shares."""
    merged = {}
    for d in parts:
        for fid, f in d.items():
            g = merged.setdefault(fid, {"members": f["members"], "stats": f["stats"], "voxels": {},
                                        "polylines": [], "isolated": []})
            assert g["members"] == f["members"] and g["stats"] == f["stats"]
            for m, cells in f["voxels"].items():
                g["voxels"].setdefault(m, []).extend(cells)
            g["polylines"].extend(f["polylines"])
            g["isolated"].extend(f["isolated"])
    return merged


@pytest.mark.parametrize("axis,normalize", [("t", True), ("z", True), ("z", False), ("t", False)])
def test_two_ranks_match_single_gpu(axis, normalize):
    import paper_1903_12294_b200 as P
    ps, fs = _dataset()
    params = _params(normalize)
    ref, rnorm, _ = P.segment(ps, fs, params)
    mm, _ = P.merge_clusters(ref.centers, 0.05)
    rfeats = _features_digest(P.build_features(ref, mm, ps, fs))
    res = _run_ranks(2, axis, normalize)
    nt = len(fs.times)
    nx, ny, nz = fs.dims
    if axis == "t":
        fl = np.concatenate([r["fl"] for r in res])
    else:
        fl = np.concatenate([r["fl"].reshape(nt, r["nz"], nx * ny) for r in res], axis=1).reshape(-1)
        assert [r["off"][2] for r in res] == [0, res[0]["nz"]]
    np.testing.assert_array_equal(fl, ref.field_labels)
    pl = np.full(len(ps), -1, np.int32)
    for r in res:
        assert np.all(pl[r["idx"]] == -1)
        pl[r["idx"]] = r["pl"]
    np.testing.assert_array_equal(pl, ref.point_labels)
    for r in res:
        assert r["it"] == ref.iterations_used
        assert r["norm"] == rnorm.to_dict()
        assert r["centers"] == [c.__dict__ for c in ref.centers]
    assert _merge_digests([r["feats"] for r in res]) == rfeats


@pytest.mark.parametrize("axis", ["t", "z"])
def test_one_rank_nccl_matches_single_gpu(axis):
    """segment_sharded + build_features_sharded through an NCCL group of one rank."""
    import torch.distributed as dist
    import paper_1903_12294_b200 as P
    from paper_1903_12294_b200.parallel import segment_sharded, shard_dataset
    from paper_1903_12294_b200.postproc import build_features_sharded
    ps, fs = _dataset(seed=12)
    params = _params(True)
    ref, rnorm, _ = P.segment(ps, fs, params)
    mm, _ = P.merge_clusters(ref.centers, 0.05)
    rfeats = _features_digest(P.build_features(ref, mm, ps, fs))
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        lps, lfs, off, gd, idx, m0 = shard_dataset(ps, fs, params.k, 0, 1, axis)
        seg, norm, _ = segment_sharded(lps, lfs, params, field_offset=off, grid_dims=gd)
        feats = build_features_sharded(seg, mm, lps, lfs, point_index=idx, field_offset=off,
                                       timestep_offset=m0, grid_dims=gd)
    finally:
        dist.destroy_process_group()
    np.testing.assert_array_equal(seg.field_labels, ref.field_labels)
    np.testing.assert_array_equal(seg.point_labels, ref.point_labels)
    assert norm == rnorm
    assert _features_digest(feats) == rfeats


def test_zslab_offset_single_process_bit_identical():
    """Two z-slabs (DeviceField.offset) emulated on one GPU pass by pass (no
    collective): per pass each slab is assigned separately, the exact partial
    sums are added through the limb encoding and the centres updated; labels and
    centres equal the whole-grid run bit for bit.  A non-trivial origin and
    spacing make the global-index cell centres matter."""
    import ctypes as C
    from paper_1903_12294_b200 import ClusterParams, _native as N, seed_centers
    from paper_1903_12294_b200.engine import (CenterState, DeviceField, DevicePoints, _run_assign,
                                              empty_state, make_params, run_device, state_struct,
                                              stream_ptr)
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device, synthetic_device
    from paper_1903_12294_b200.model import interval_distances
    from paper_1903_12294_b200.parallel import select_points_for_slab, slab_bin_ranges, zbin_slabs, cell_centres
    lib = N.load()
    dims, nt = (20, 16, 40), 6
    fld0, pts, _ = synthetic_device(dims, nt, 500, seed=23)
    origin, spacing = np.array([0.3, -7.1, 1e3 + 0.1]), np.array([0.7, 1.3, 0.1])
    fld = DeviceField(dims, origin, spacing, fld0.times, fld0.values)
    pts.xyz.mul_(torch.as_tensor(spacing, device="cuda")).add_(torch.as_tensor(origin, device="cuda"))
    normalize_device(pts, fld, True)
    ext = domain_extent_device(pts, fld)
    params = ClusterParams(k=(3, 3, 5, 2), w_d=0.8, eps_c=1e-12, max_iterations=4)
    ref = run_device(pts, fld, ext, params)
    ref_state = CenterState.from_device(ref.state)
    K = params.k_total
    C_ = interval_distances(ext, params.k)
    slabs = zbin_slabs(dims[2], origin[2], spacing[2], ext.mins[2], C_[2], params.k[2], 2)
    ranges = slab_bin_ranges(cell_centres(dims[2], origin[2], spacing[2]), ext.mins[2], C_[2],
                             params.k[2], slabs)
    plane = dims[0] * dims[1]
    vals = fld.values.reshape(nt, dims[2], plane)
    parts = []
    for (k0, k1), (b0, b1) in zip(slabs, ranges):
        sel = select_points_for_slab(pts.xyz[:, 2], ext.mins[2], C_[2], params.k[2], b0, b1)
        parts.append((DevicePoints(pts.xyz[sel].contiguous(), pts.t[sel].contiguous(),
                                   pts.value[sel].contiguous()),
                      DeviceField((dims[0], dims[1], k1 - k0), origin, spacing, fld.times,
                                  vals[:, k0:k1].contiguous().reshape(-1), (0, 0, k0)), sel))
    assert all(p[1].dims[2] > 0 for p in parts)
    state = CenterState.from_seeds(seed_centers(ext, params.k)).to_device()
    for it in range(params.max_iterations + 1):
        prm = make_params(ext.mins, C_, params, (1.0, 0.0, 0.0) if it == 0 else None)
        limbs, labs = None, []
        for sp, sf, _ in parts:
            pl, fl, acc = _run_assign(sp, sf, state, prm, K)
            lb = torch.empty(K * 8 * 3, dtype=torch.int64, device=acc.device)
            N.check(lib.mfseg_acc_to_limbs(N.ptr(acc), K * 8, N.ptr(lb), stream_ptr()), "limbs")
            limbs = lb if limbs is None else limbs + lb
            labs.append((pl, fl))
        acc = torch.empty((K, N.ACC_WORDS), dtype=torch.int64, device=limbs.device)
        N.check(lib.mfseg_limbs_to_acc(N.ptr(limbs), K * 8, N.ptr(acc), stream_ptr()), "acc")
        new = empty_state(K)
        conv, delta = C.c_int32(0), C.c_double(0.0)
        N.check(lib.mfseg_update_centers(K, N.ptr(acc), state_struct(state), state_struct(new),
                                         params.eps_c, C.byref(conv), C.byref(delta), stream_ptr()),
                "update")
        state = new
        if it > 0 and conv.value:
            break
    fl = torch.cat([labs[r][1].reshape(nt, -1, plane) for r in range(2)], dim=1).reshape(-1)
    assert torch.equal(fl, ref.field_labels)
    pl = torch.empty_like(ref.point_labels)
    for r in range(2):
        pl[parts[r][2]] = labs[r][0]
    assert torch.equal(pl, ref.point_labels)
    st = CenterState.from_device(state)
    np.testing.assert_array_equal(st.loc, ref_state.loc)
    np.testing.assert_array_equal(st.fval, ref_state.fval)


@pytest.mark.parametrize("config", ["small", "smallz"])
def test_bench_two_ranks_functional(config):
    """bench.py's multi-rank path (rank slabs generated in place, sharded
    normalisation + extent, per-pass exchange, e2e through segment_sharded) runs
    end to end under torchrun with two ranks on one GPU (gloo: host-side
    exchange) and prints one JSON line for the whole job."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MFSEG_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                          str(_free_port()), os.path.join(root, "bench.py"), "--gpus", "2",
                          "--config", config, "--steps", "2", "--warmup", "3"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["voxel_timesteps"] == 64 * 64 * 32 * 16
