"""Parity of the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.

Bars (written in the asserts):
  * labels, counts, ids, merge maps, voxel lists, bboxes: bit-exact;
  * centre locations/values: within 1e-12 relative of the reference (exact
    128-bit sums vs numpy's sequential fp64 sums; north_star allows 1e-5);
  * feature mean/std: within 1e-9 relative to the value scale (north_star 1e-5).
"""
import numpy as np
import pytest
import torch

from golden_io import Case, names

from paper_1903_12294_b200 import _native as N

pytestmark = pytest.mark.gpu

RUNS = names("run_")
ASSIGNS = names("assign_")
CENTER_RTOL = 1e-12


def pkg():
    import paper_1903_12294_b200 as P
    return P


def _points(case):
    P = pkg()
    if case["in_p_t"].size == 0:
        return P.PointSet.empty()
    return P.PointSet(case["in_p_traj_id"], case["in_p_t"], case["in_p_xyz"].reshape(-1, 3),
                      case["in_p_value"])


def _field(case):
    P = pkg()
    dims, origin, spacing, times, values = case.field
    if values.size == 0:
        return P.FieldSet.empty()
    return P.FieldSet(dims, origin, spacing, times, values.reshape(len(times), -1))


def _extent(case):
    P = pkg()
    e = case.meta["extent"]
    return P.DomainExtent.from_dict(e)


def _params(case):
    P = pkg()
    return P.ClusterParams.from_dict(case.meta["params"])


def _state(case, prefix):
    P = pkg()
    return P.CenterState(case[prefix + "loc"].copy(), case[prefix + "pval"].copy(),
                         case[prefix + "fval"].copy(), case[prefix + "has_p"].copy(),
                         case[prefix + "has_f"].copy(), case[prefix + "n_points"].copy(),
                         case[prefix + "n_fields"].copy(), case[prefix + "dormant"].copy())


def _close(got, want, rtol, scale=1.0):
    """|got - want| <= rtol * max(|want|, scale): relative, except near zero where
    sums of O(scale) terms cancel (e.g. a mean of noise around 0)."""
    got, want = np.asarray(got, float), np.asarray(want, float)
    assert got.shape == want.shape
    both_nan = np.isnan(got) & np.isnan(want)
    ok = both_nan | (np.abs(got - want) <= rtol * np.maximum(np.abs(want), scale))
    assert ok.all(), (got[~ok][:5], want[~ok][:5])


@pytest.mark.parametrize("name", ASSIGNS)
def test_assign_iteration_bit_exact(name):
    P = pkg()
    case = Case(name)
    params = _params(case)
    ext = _extent(case)
    C = P.interval_distances(ext, params.k)
    cs = _state(case, "in_c_")
    grid = P.CenterGrid(cs.loc, ext, C, params.k)
    pl, fl = P.assign_iteration(_points(case), _field(case), None, cs, grid, params, C)
    np.testing.assert_array_equal(pl, case["out_point_labels"])
    np.testing.assert_array_equal(fl, case["out_field_labels"])
    assert pl.dtype == np.int64 and fl.dtype == np.int64


@pytest.mark.parametrize("name", ASSIGNS)
def test_accumulate_update_converge(name):
    P = pkg()
    case = Case(name)
    K = len(case["in_c_loc"])
    sums = P.accumulate(case["out_point_labels"], _points(case), case["out_field_labels"],
                        _field(case), None, K)
    for nm, got in zip(("sums", "psum", "fsum"), sums[:3]):
        _close(got, case[f"out_acc_{nm}"], 1e-13)
    np.testing.assert_array_equal(sums[3], case["out_acc_n_p"])
    np.testing.assert_array_equal(sums[4], case["out_acc_n_f"])
    # update from the reference's own sums: identical arithmetic -> bit-exact
    old = _state(case, "in_c_")
    new = P.update_centers(old, *(case[f"out_acc_{n}"] for n in ("sums", "psum", "fsum", "n_p", "n_f")))
    for f in ("loc", "pval", "fval", "has_p", "has_f", "n_points", "n_fields", "dormant"):
        np.testing.assert_array_equal(getattr(new, f), case[f"out_new_{f}"], err_msg=f)
    assert P.has_converged(old, new, case.meta["params"]["eps_c"]) == case.meta["converged"]
    assert P.max_center_delta(old, new) == case.meta["max_delta"]


@pytest.mark.parametrize("name", RUNS)
def test_run_matches_reference(name):
    P = pkg()
    case = Case(name)
    params = _params(case)
    pts = _points(case) if case["in_p_t"].size else None
    fld = _field(case) if case["in_f_values"].size else None
    prog = []
    seg = P.run(pts, fld, _extent(case), params, progress=lambda i, d: prog.append((i, d)))
    np.testing.assert_array_equal(seg.point_labels, case["out_point_labels"])
    np.testing.assert_array_equal(seg.field_labels, case["out_field_labels"])
    assert seg.point_labels.dtype == np.int32
    assert seg.iterations_used == case.meta["iterations_used"]
    assert seg.converged == case.meta["converged"]
    ids = np.array([c.id for c in seg.centers])
    np.testing.assert_array_equal(ids, case["out_c_id"])
    _close([[c.x_c, c.y_c, c.z_c, c.t_c] for c in seg.centers], case["out_c_loc"], CENTER_RTOL)
    _close([np.nan if c.p_c is None else c.p_c for c in seg.centers], case["out_c_p_c"], CENTER_RTOL)
    _close([np.nan if c.f_c is None else c.f_c for c in seg.centers], case["out_c_f_c"], CENTER_RTOL)
    np.testing.assert_array_equal([c.n_points for c in seg.centers], case["out_c_n_points"])
    np.testing.assert_array_equal([c.n_fields for c in seg.centers], case["out_c_n_fields"])
    assert [i for i, _ in prog] == [i for i, _ in case.meta["progress"]]
    got_d = np.array([d for _, d in prog])
    want_d = np.array([d for _, d in case.meta["progress"]])
    assert np.all(np.abs(got_d - want_d) <= 1e-6 * np.abs(want_d) + 1e-12)


def test_pipeline_segment_frontend_fixture():
    """Raw inputs -> device normalize -> extent -> run: the reference's recorded
    service responses (frontend fixtures) within 1e-12."""
    P = pkg()
    case = Case("run_slab2_frontend")
    params = _params(case)
    raw_p = P.PointSet(case["in_p_traj_id"], case["in_p_t"], case["in_p_xyz"].reshape(-1, 3),
                       case["in_raw_p_value"])
    dims, origin, spacing, times, _ = case.field
    raw_f = P.FieldSet(dims, origin, spacing, times, case["in_raw_f_values"])
    seg, norm, _ = P.segment(raw_p, raw_f, params)
    want = case.meta["normalization"]
    assert norm.to_dict() == want
    assert seg.extent.to_dict() == case.meta["extent"]
    np.testing.assert_array_equal(seg.point_labels, case["out_point_labels"])
    np.testing.assert_array_equal(seg.field_labels, case["out_field_labels"])
    fx = case.meta["frontend_fixture"]
    for c, w in zip(seg.centers, fx["centers_all"]):
        _close([c.x_c, c.y_c, c.z_c, c.t_c, c.p_c, c.f_c],
               [w["x_c"], w["y_c"], w["z_c"], w["t_c"], w["p_c"], w["f_c"]], CENTER_RTOL)
        assert (c.n_points, c.n_fields) == (w["n_points"], w["n_fields"])
    mm, merged = P.merge_clusters(seg.centers, 2.0)
    assert {str(k): v for k, v in mm.items()} == fx["merge_all"]["merge_map"]
    w = fx["merge_all"]["centers"][0]
    _close([merged[0].x_c, merged[0].y_c, merged[0].z_c, merged[0].t_c, merged[0].p_c,
            merged[0].f_c], [w["x_c"], w["y_c"], w["z_c"], w["t_c"], w["p_c"], w["f_c"]],
           CENTER_RTOL)


def _rows(case, prefix):
    P = pkg()
    out = []
    for i, loc, pc, fc, n_p, n_f in zip(case[prefix + "id"], case[prefix + "loc"],
                                        case[prefix + "p_c"], case[prefix + "f_c"],
                                        case[prefix + "n_points"], case[prefix + "n_fields"]):
        out.append(P.ClusterCenter(int(i), *map(float, loc), None if np.isnan(pc) else float(pc),
                                   None if np.isnan(fc) else float(fc), int(n_p), int(n_f)))
    return out


@pytest.mark.parametrize("name", RUNS)
def test_merge_bit_exact(name):
    P = pkg()
    case = Case(name)
    rows = _rows(case, "out_c_")
    for key in case.meta["merges"]:
        mm, merged = P.merge_clusters(rows, float(key))
        assert [mm[int(i)] for i in case[f"merge_{key}_ids"]] == list(case[f"merge_{key}_rep"])
        want = _rows(case, f"merge_{key}_c_")
        assert merged == want      # dataclass equality: every field bit-identical


@pytest.mark.parametrize("name", [n for n in RUNS if n not in ("run_blob_k256", "run_stripes_lo",
                                                               "run_stripes_hi")])
def test_features_match_reference(name):
    P = pkg()
    case = Case(name)
    rows = _rows(case, "out_c_")
    seg = P.Segmentation(case["out_point_labels"], case["out_field_labels"], rows,
                         _params(case), _extent(case), case.meta["iterations_used"],
                         case.meta["converged"])
    pts, fld = _points(case), _field(case)
    for key, want in case.meta["features"].items():
        mm = None if key == "identity" else P.merge_clusters(rows, float(key))[0]
        got = P.build_features(seg, mm, pts, fld)
        assert [f.id for f in got] == [w["id"] for w in want]
        for g, w in zip(got, want):
            assert g.member_clusters == w["member_clusters"]
            assert [list(map(int, x)) for x in g.polylines] == w["polylines"]
            assert g.isolated_points == w["isolated_points"]
            assert {str(m): list(map(int, c)) for m, c in sorted(g.voxels.items())} == w["voxels"]
            s = g.stats.to_dict()
            for k in ("bbox_min", "bbox_max", "n_points", "n_fields"):
                assert s[k] == w["stats"][k], (k, s[k], w["stats"][k])
            for k in ("p_mean", "p_std", "f_mean", "f_std"):
                if w["stats"][k] is None:
                    assert s[k] is None
                else:
                    scale = max(abs(w["stats"][k.replace("std", "mean")] or 0.0), 1.0)
                    assert abs(s[k] - w["stats"][k]) <= 1e-9 * scale, (k, s[k], w["stats"][k])


def test_link_index_matches_reference():
    P = pkg()
    case = Case("link_blob")
    li = P.build_link_index(_field(case), _points(case))
    keys = list(li.buckets)
    np.testing.assert_array_equal(np.array(keys).reshape(-1, 4), case["out_keys"])
    np.testing.assert_array_equal([len(li.buckets[k]) for k in keys], case["out_sizes"])
    np.testing.assert_array_equal(np.concatenate([li.buckets[k] for k in keys]),
                                  case["out_members"])


def test_link_index_rejects_outside_points():
    P = pkg()
    fs = P.FieldSet((4, 4, 4), np.zeros(3), np.ones(3), np.array([0.0, 1.0, 2.0]), np.zeros((3, 64)))
    ps = P.PointSet(np.array([0]), np.array([0.0]), np.array([[9.0, 0.5, 0.5]]), np.array([1.0]))
    with pytest.raises(P.IngestError):
        P.build_link_index(fs, ps)


# ------------------------------------------------------------------ synthetic, vs the C oracle

def _synthetic(dims, nt, ntraj, seed, dyadic, noise=0.05, n_blobs=5):
    from paper_1903_12294_b200.ingest import synthetic_device
    return synthetic_device(dims, nt, ntraj, seed=seed, noise=noise, n_blobs=n_blobs, dyadic=dyadic)


@pytest.mark.parametrize("dyadic", [False, True])
def test_synthetic_generator_matches_numpy_mirror(dyadic):
    from oracle import synth
    dims, nt, ntraj = (20, 12, 9), 5, 50
    fld, pts, tid = _synthetic(dims, nt, ntraj, seed=7, dyadic=dyadic)
    np.testing.assert_array_equal(fld.values.cpu().numpy().reshape(nt, -1),
                                  synth.field(dims, nt, seed=7, n_blobs=5, dyadic=dyadic))
    t_id, t, xyz, v = synth.points(dims, nt, ntraj, seed=7, n_blobs=5, dyadic=dyadic)
    np.testing.assert_array_equal(tid.cpu().numpy(), t_id)
    np.testing.assert_array_equal(pts.t.cpu().numpy(), t)
    np.testing.assert_array_equal(pts.xyz.cpu().numpy(), xyz)
    np.testing.assert_array_equal(pts.value.cpu().numpy(), v)


@pytest.mark.parametrize("dyadic,k,seed", [(True, (6, 5, 4, 3), 1), (False, (6, 5, 4, 3), 2),
                                           (False, (8, 8, 4, 4), 3), (True, (3, 3, 3, 2), 4)])
def test_run_vs_c_oracle(dyadic, k, seed):
    """Full runs on the counter-based generator vs the C restatement."""
    from oracle import c_oracle
    from oracle import mfseg_oracle as O
    from paper_1903_12294_b200 import ClusterParams
    from paper_1903_12294_b200.engine import CenterState, run_device
    from paper_1903_12294_b200.ingest import domain_extent_device
    dims, nt, ntraj = (40, 32, 20), 8, 1500
    fld, pts, _ = _synthetic(dims, nt, ntraj, seed, dyadic)
    ext = domain_extent_device(pts, fld)
    params = ClusterParams(k=k, w_d=0.7, eps_c=1e-12, max_iterations=6, normalize=False)
    r = run_device(pts, fld, ext, params)
    floc = O.field_locations(dims, np.zeros(3), np.ones(3), np.arange(nt, dtype=float))
    ref = c_oracle.run(np.column_stack([pts.xyz.cpu().numpy(), pts.t.cpu().numpy()]),
                       pts.value.cpu().numpy(), floc, fld.values.cpu().numpy(), ext.mins,
                       ext.maxs, k, c_f=1.0, w_d=0.7, w_p=1.0, w_f=1.0, eps_c=1e-12,
                       max_iterations=6)
    np.testing.assert_array_equal(r.field_labels.cpu().numpy(), ref["field_labels"])
    np.testing.assert_array_equal(r.point_labels.cpu().numpy(), ref["point_labels"])
    assert r.iterations_used == ref["iterations_used"]
    st = CenterState.from_device(r.state)
    np.testing.assert_array_equal(st.n_points, ref["n_points"])
    np.testing.assert_array_equal(st.n_fields, ref["n_fields"])
    if dyadic:   # every sum exact in both -> bit-identical centres
        np.testing.assert_array_equal(st.loc, ref["loc"])
        np.testing.assert_array_equal(st.pval, ref["pval"])
        np.testing.assert_array_equal(st.fval, ref["fval"])
    else:
        _close(st.loc, ref["loc"], CENTER_RTOL)
        _close(st.pval, ref["pval"], CENTER_RTOL)


def test_stranded_and_crowded_bins_vs_oracle():
    """Heavily drifted, crowded centres: many stranded samples and long
    candidate lists (> one 256-candidate chunk) through the fallback path."""
    from oracle import c_oracle
    from oracle import mfseg_oracle as O
    P = pkg()
    rng = np.random.default_rng(5)
    dims, nt = (30, 20, 10), 6
    fs = P.FieldSet(dims, np.zeros(3), np.ones(3), np.arange(nt, dtype=float),
                    rng.random((nt, int(np.prod(dims)))))
    n = 4000
    loc = rng.random((n, 4)) * [30, 20, 10, 5]
    ps = P.PointSet(np.arange(n), loc[:, 3].copy(), loc[:, :3].copy(), rng.random(n))
    ext = P.DomainExtent(0, 30, 0, 20, 0, 10, 0, 5)
    params = P.ClusterParams(k=(10, 8, 4, 3), w_d=1.0, w_p=0.8, w_f=0.5)
    K = params.k_total
    C = P.interval_distances(ext, params.k)
    seeds = P.seed_centers(ext, params.k)
    cs = P.CenterState.from_seeds(seeds + rng.uniform(-2.5, 2.5, (K, 4)) * C)
    cs.loc[:300] = cs.loc[0] + rng.uniform(-0.2, 0.2, (300, 4)) * C     # 300 centres in one bin
    cs.pval = np.where(rng.random(K) < 0.7, rng.random(K), np.nan)
    cs.fval = np.where(rng.random(K) < 0.7, rng.random(K), np.nan)
    cs.has_p, cs.has_f = ~np.isnan(cs.pval), ~np.isnan(cs.fval)
    grid = P.CenterGrid(cs.loc, ext, C, params.k)
    pl, fl = P.assign_iteration(ps, fs, None, cs, grid, params, C)
    floc = O.field_locations(dims, np.zeros(3), np.ones(3), fs.times)
    epl = c_oracle.assign(ps.loc4, ps.value, cs.loc, cs.pval, cs.has_p, ext.mins, C, params.k,
                          params.w_p, params.w_d, params.c_f)
    efl = c_oracle.assign(floc, fs.flat_values(), cs.loc, cs.fval, cs.has_f, ext.mins, C,
                          params.k, params.w_f, params.w_d, params.c_f)
    np.testing.assert_array_equal(pl, epl)
    np.testing.assert_array_equal(fl, efl)


def test_empty_kinds_and_errors():
    P = pkg()
    ext = P.DomainExtent(0, 10, 0, 10, 0, 10, 0, 4)
    with pytest.raises(ValueError):
        P.run(None, None, ext, P.ClusterParams())
    rng = np.random.default_rng(2)
    loc = rng.random((50, 4)) * [10, 10, 10, 4]
    pts = P.PointSet(np.arange(50), loc[:, 3].copy(), loc[:, :3].copy(), rng.random(50))
    seg = P.run(pts, None, ext, P.ClusterParams(k=(1, 1, 1, 1), normalize=False))
    assert seg.converged and seg.iterations_used <= 2
    c = seg.centers[0]
    np.testing.assert_allclose(c.loc4, pts.loc4.mean(axis=0), rtol=1e-14)
    assert c.f_c is None and len(seg.field_labels) == 0


def test_labels_deterministic_across_reruns():
    from paper_1903_12294_b200 import ClusterParams
    from paper_1903_12294_b200.engine import CenterState, run_device
    from paper_1903_12294_b200.ingest import domain_extent_device
    fld, pts, _ = _synthetic((48, 40, 24), 6, 4000, 11, False)
    ext = domain_extent_device(pts, fld)
    params = ClusterParams(k=(6, 5, 3, 2), w_d=0.5, eps_c=1e-12, max_iterations=5)
    a = run_device(pts, fld, ext, params)
    sa = CenterState.from_device(a.state)
    la, lb = a.field_labels.clone(), a.point_labels.clone()
    b = run_device(pts, fld, ext, params)
    sb = CenterState.from_device(b.state)
    assert torch.equal(la, b.field_labels) and torch.equal(lb, b.point_labels)
    np.testing.assert_array_equal(sa.loc, sb.loc)


def test_time_slab_sharding_bit_identical():
    """Two 'ranks' emulated on one GPU: per pass each time slab is assigned
    separately, the exact 128-bit partial sums are summed through the limb
    encoding (as the NCCL exchange does), and the centres updated.  Labels and
    centres must equal the single-GPU run bit for bit."""
    import ctypes as C
    from paper_1903_12294_b200 import ClusterParams, _native as N
    from paper_1903_12294_b200.engine import (DeviceField, DevicePoints, CenterState, _run_assign,
                                              empty_state, make_params, run_device, state_struct,
                                              stream_ptr)
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
    from paper_1903_12294_b200.model import interval_distances
    from paper_1903_12294_b200.parallel import time_slab
    lib = N.load()
    dims, nt = (32, 24, 16), 8
    fld, pts, _ = _synthetic(dims, nt, 2000, 21, False)
    normalize_device(pts, fld, True)
    ext = domain_extent_device(pts, fld)
    params = ClusterParams(k=(4, 4, 4, 4), w_d=0.8, eps_c=1e-12, max_iterations=4)
    ref = run_device(pts, fld, ext, params)
    ref_state = CenterState.from_device(ref.state)
    K = params.k_total
    C_ = interval_distances(ext, params.k)
    ncell = int(np.prod(dims))
    slabs = []
    for r in range(2):
        m0, m1 = time_slab(r, 2, nt)
        sel = (pts.t >= m0) & (pts.t < m1)
        slabs.append((DevicePoints(pts.xyz[sel].contiguous(), pts.t[sel].contiguous(),
                                   pts.value[sel].contiguous()),
                      DeviceField(fld.dims, fld.origin, fld.spacing, fld.times[m0:m1].clone(),
                                  fld.values[m0 * ncell:m1 * ncell].clone()),
                      sel))
    seeds = CenterState.from_seeds(P_seed(ext, params.k))
    state = seeds.to_device()
    for it in range(params.max_iterations + 1):
        w = (1.0, 0.0, 0.0) if it == 0 else None
        prm = make_params(ext.mins, C_, params, w)
        limbs = None
        labs = []
        for sp, sf, _ in slabs:
            pl, fl, acc = _run_assign(sp, sf, state, prm, K)
            lb = torch.empty(K * 8 * 3, dtype=torch.int64, device=acc.device)
            N.check(lib.mfseg_acc_to_limbs(N.ptr(acc), K * 8, N.ptr(lb), stream_ptr()), "limbs")
            limbs = lb if limbs is None else limbs + lb
            labs.append((pl, fl))
        acc = torch.empty((K, N.ACC_WORDS), dtype=torch.int64, device=limbs.device)
        N.check(lib.mfseg_limbs_to_acc(N.ptr(limbs), K * 8, N.ptr(acc), stream_ptr()), "from limbs")
        new = empty_state(K)
        conv, delta = C.c_int32(0), C.c_double(0.0)
        N.check(lib.mfseg_update_centers(K, N.ptr(acc), state_struct(state), state_struct(new),
                                         params.eps_c, C.byref(conv), C.byref(delta), stream_ptr()),
                "update")
        state = new
        if it > 0 and conv.value:
            break
    field_labels = torch.cat([labs[0][1], labs[1][1]])
    assert torch.equal(field_labels, ref.field_labels)
    point_labels = torch.empty_like(ref.point_labels)
    point_labels[slabs[0][2]] = labs[0][0]
    point_labels[slabs[1][2]] = labs[1][0]
    assert torch.equal(point_labels, ref.point_labels)
    st = CenterState.from_device(state)
    np.testing.assert_array_equal(st.loc, ref_state.loc)
    np.testing.assert_array_equal(st.pval, ref_state.pval)
    np.testing.assert_array_equal(st.fval, ref_state.fval)


def P_seed(ext, k):
    from paper_1903_12294_b200 import seed_centers
    return seed_centers(ext, k)


def test_limb_kernels_match_python_encoding():
    from paper_1903_12294_b200 import _native as N
    from paper_1903_12294_b200.engine import stream_ptr
    lib = N.load()
    rng = np.random.default_rng(3)
    vals = [int(x) * (1 << 50) + int(y) for x, y in zip(rng.integers(-2**60, 2**60, 64),
                                                         rng.integers(0, 2**50, 64))]
    lo = [(v & ((1 << 64) - 1)) for v in vals]
    hi = [((v >> 64) & ((1 << 64) - 1)) for v in vals]
    acc = torch.tensor(np.array([x for pair in zip(lo, hi) for x in pair], dtype=np.uint64).view(np.int64),
                       device="cuda")
    limbs = torch.empty(64 * 3, dtype=torch.int64, device="cuda")
    N.check(lib.mfseg_acc_to_limbs(N.ptr(acc), 64, N.ptr(limbs), stream_ptr()), "limbs")
    L = limbs.cpu().numpy().tolist()
    for i, v in enumerate(vals):
        assert L[3 * i] + (L[3 * i + 1] << 42) + (L[3 * i + 2] << 84) == v
    back = torch.empty_like(acc)
    N.check(lib.mfseg_limbs_to_acc(N.ptr(limbs), 64, N.ptr(back), stream_ptr()), "acc")
    assert torch.equal(back, acc)


def _oracle_labels(ps, fs, cs, ext, C, params):
    """The C oracle's windowed assignment (engine.py:164-218) of both kinds."""
    from oracle import c_oracle
    ploc = np.column_stack([ps.xyz, ps.t])
    pl = c_oracle.assign(ploc, ps.value, cs.loc, cs.pval, cs.has_p, ext.mins, C, params.k,
                         params.w_p, params.w_d, params.c_f)
    fl = c_oracle.assign_field(fs.dims, fs.origin, fs.spacing, fs.times, fs.values, cs.loc,
                               cs.fval, cs.has_f, ext.mins, C, params.k, params.w_f, params.w_d,
                               params.c_f)
    return pl, fl


@pytest.mark.parametrize("w_d,seed", [(1.0, 21), (0.15, 22)])
def test_assign_drifted_centres_vs_oracle(w_d, seed):
    """The field (block culling, dominance, packed-key screen) and point kernels
    against the C oracle on drifted centres with and without values: one
    assignment pass over ~6M voxel-timesteps and 150k points, labels bit-exact.
    A small w_d makes the value term large (dominance's value bound)."""
    P = pkg()
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
    dims, nt, ntraj = (96, 80, 48), 16, 10000
    fld, pts, _ = _synthetic(dims, nt, ntraj, seed, False)
    normalize_device(pts, fld, True)
    ext = domain_extent_device(pts, fld)
    params = P.ClusterParams(k=(6, 5, 3, 4), w_d=w_d, w_p=1.0, w_f=1.0)
    rng = np.random.default_rng(seed)
    K = params.k_total
    C = P.interval_distances(ext, params.k)
    cs = P.CenterState.from_seeds(P.seed_centers(ext, params.k) + rng.uniform(-0.45, 0.45, (K, 4)) * C)
    cs.pval = np.where(rng.random(K) < 0.8, rng.random(K), np.nan)
    cs.fval = np.where(rng.random(K) < 0.8, rng.random(K), np.nan)
    cs.has_p, cs.has_f = ~np.isnan(cs.pval), ~np.isnan(cs.fval)
    grid = P.CenterGrid(cs.loc, ext, C, params.k)
    fs = P.FieldSet(dims, np.zeros(3), np.ones(3), fld.times.cpu().numpy(),
                    fld.values.cpu().numpy().reshape(nt, -1))
    ps = P.PointSet(np.zeros(pts.n, np.int64), pts.t.cpu().numpy(), pts.xyz.cpu().numpy(),
                    pts.value.cpu().numpy())
    pl, fl = P.assign_iteration(ps, fs, None, cs, grid, params, C)
    want_p, want_f = _oracle_labels(ps, fs, cs, ext, C, params)
    np.testing.assert_array_equal(fl, want_f)
    np.testing.assert_array_equal(pl, want_p)


@pytest.mark.parametrize("seed", [31, 32])
def test_points_on_bin_and_subcell_edges_vs_oracle(seed):
    """Point sort keys take the bin from a reciprocal product and divide exactly
    only near a sub-cell edge (k_point_keys): points placed exactly on bin and
    eighth-of-bin edges of a non-dyadic extent, and one ulp either side, are
    binned and labelled like the C oracle's fl((x - min) / C)."""
    P = pkg()
    rng = np.random.default_rng(seed)
    ext = P.DomainExtent(0.1, 1.37, -0.3, 0.71, 0.05, 0.93, 3.0, 17.7)
    params = P.ClusterParams(k=(7, 5, 3, 6), w_d=1.0, w_p=1.0, w_f=1.0)
    C = P.interval_distances(ext, params.k)
    mins, maxs = ext.mins, ext.maxs
    n = 60000
    loc = np.empty((n, 4))
    for d in range(4):
        j = rng.integers(0, 8 * params.k[d] + 1, n)
        x = mins[d] + j * (C[d] / 8.0)
        step = rng.integers(-1, 2, n)
        x = np.where(step < 0, np.nextafter(x, -np.inf), np.where(step > 0, np.nextafter(x, np.inf), x))
        loc[:, d] = np.clip(x, mins[d], maxs[d])
    ps = P.PointSet(np.arange(n, dtype=np.int64) // 8, loc[:, 3].copy(), loc[:, :3].copy(), rng.random(n))
    dims, nt = (5, 4, 3), 2
    fs = P.FieldSet(dims, np.array([0.2, -0.2, 0.1]), np.array([0.25, 0.2, 0.25]), np.array([4.0, 9.0]),
                    rng.random((nt, int(np.prod(dims)))))
    K = params.k_total
    cs = P.CenterState.from_seeds(P.seed_centers(ext, params.k) + rng.uniform(-0.45, 0.45, (K, 4)) * C)
    cs.pval = np.where(rng.random(K) < 0.8, rng.random(K), np.nan)
    cs.fval = np.where(rng.random(K) < 0.8, rng.random(K), np.nan)
    cs.has_p, cs.has_f = ~np.isnan(cs.pval), ~np.isnan(cs.fval)
    grid = P.CenterGrid(cs.loc, ext, C, params.k)
    pl, fl = P.assign_iteration(ps, fs, None, cs, grid, params, C)
    want_p, want_f = _oracle_labels(ps, fs, cs, ext, C, params)
    np.testing.assert_array_equal(pl, want_p)
    np.testing.assert_array_equal(fl, want_f)


@pytest.mark.parametrize("opts", [dict(multi_cap=0), dict(multi_cap=37), dict(flags=2),
                                  dict(flags=1), dict(flags=16), dict(flags=32), dict(flags=64),
                                  dict(flags=256)])
def test_field_brick_queue_paths_agree(opts):
    """k_field_assign5 queues multi-candidate bricks for k_field_screen; a full
    queue (capacity 0 or 37 items) sends the rest to the exact per-sample path
    (k_deferred), debug flag 2 resolves every queued sample in exact fp64 and
    flag 1 disables culling and dominance (most bricks then exceed the
    16-candidate queue limit); flag 16 recomputes the blocks whose candidates
    did not change since the last pass, flag 32 keeps only exact reuse, flag 64
    labels the initial pass without the interior-block / chunk shortcut.  A 6-pass run: labels and
    centre positions bit-identical (integer sums), field means within fp64
    rounding (the value
    sums are rounded per record or per sample depending on the path)."""
    P = pkg()
    dims, nt, ntraj = (64, 48, 40), 8, 2000
    fld, pts, _ = _synthetic(dims, nt, ntraj, 31, False)
    fs = P.FieldSet(dims, np.zeros(3), np.ones(3), fld.times.cpu().numpy(),
                    fld.values.cpu().numpy().reshape(nt, -1))
    ps = P.PointSet(np.zeros(pts.n, np.int64), pts.t.cpu().numpy(), pts.xyz.cpu().numpy(),
                    pts.value.cpu().numpy())
    ext = P.domain_extent(ps, fs)
    params = P.ClusterParams(k=(5, 4, 3, 2), w_d=0.3, max_iterations=5, eps_c=1e-12)
    a = P.run(ps, fs, ext, params)
    with N.debug_options(**opts):
        b = P.run(ps, fs, ext, params)
    np.testing.assert_array_equal(a.field_labels, b.field_labels)
    np.testing.assert_array_equal(a.point_labels, b.point_labels)
    assert [c.id for c in a.centers] == [c.id for c in b.centers]
    for ca, cb in zip(a.centers, b.centers):
        assert (ca.x_c, ca.y_c, ca.z_c, ca.t_c) == (cb.x_c, cb.y_c, cb.z_c, cb.t_c)
        assert (ca.n_points, ca.n_fields, ca.p_c) == (cb.n_points, cb.n_fields, cb.p_c)
        assert (ca.f_c is None) == (cb.f_c is None)
        if ca.f_c is not None:
            assert ca.f_c == pytest.approx(cb.f_c, rel=1e-12, abs=1e-15)


@pytest.mark.parametrize("c_f,k,iters", [(1.0, (8, 6, 4, 6), 1), (0.37, (16, 12, 8, 6), 1),
                                          (2.5, (5, 7, 3, 4), 2)])
def test_initial_pass_shortcut_is_exact(c_f, k, iters):
    """The initial pass labels field blocks and point chunks lying inside their
    bin (margin 2^-20 bin widths) with the bin's own seed without any candidate
    work: labels and centres must equal the full windowed assignment (debug flag
    NO_SEEDS_FAST), including the samples on bin faces (integer grid, bins of
    whole cells) that the shortcut must leave to the exact path."""
    P = pkg()
    from paper_1903_12294_b200.engine import run_device
    from paper_1903_12294_b200.ingest import domain_extent_device
    dims, nt, ntraj = (96, 80, 48), 18, 20000
    fld, pts, _ = _synthetic(dims, nt, ntraj, 17, False, n_blobs=2)
    ext = domain_extent_device(pts, fld)
    params = P.ClusterParams(k=k, c_f=c_f, eps_c=1e-12, max_iterations=iters)
    a = run_device(pts, fld, ext, params)
    with N.debug_options(N.DEBUG_NO_SEEDS_FAST):
        b = run_device(pts, fld, ext, params)
    assert torch.equal(a.field_labels, b.field_labels)
    assert torch.equal(a.point_labels, b.point_labels)
    sa, sb = P.CenterState.from_device(a.state), P.CenterState.from_device(b.state)
    np.testing.assert_array_equal(np.asarray(sa.loc), np.asarray(sb.loc))
    np.testing.assert_array_equal(np.asarray(sa.fval), np.asarray(sb.fval))
    np.testing.assert_array_equal(np.asarray(sa.pval), np.asarray(sb.pval))


@pytest.mark.parametrize("c_f,nz,kz", [(1.0, 1, 1), (0.45, 1, 1), (2.0, 1, 1), (1.0, 1, 2)])
def test_thin_field_time_blocks_are_exact(c_f, nz, kz):
    """Fields of one z plane and one z bin run the field kernels with their z axis
    over the timesteps (FieldArgs.swap_zt): labels, positions and point values
    equal the z-axis blocking (debug flag NO_ZT_SWAP) bit for bit, field values
    within fp64 rounding, for several time scales c_f; a second z bin (k_z = 2)
    keeps the z blocking."""
    P = pkg()
    from paper_1903_12294_b200.engine import run_device
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
    dims, nt, ntraj = (120, 72, nz), 37, 15000
    fld, pts, _ = _synthetic(dims, nt, ntraj, 23, False, n_blobs=3)
    normalize_device(pts, fld, True)
    ext = domain_extent_device(pts, fld)
    params = P.ClusterParams(k=(7, 5, kz, 6), c_f=c_f, eps_c=1e-12, max_iterations=6)
    a = run_device(pts, fld, ext, params)
    with N.debug_options(N.DEBUG_NO_ZT_SWAP):
        b = run_device(pts, fld, ext, params)
    assert a.iterations_used == b.iterations_used
    assert torch.equal(a.field_labels, b.field_labels)
    assert torch.equal(a.point_labels, b.point_labels)
    sa, sb = P.CenterState.from_device(a.state), P.CenterState.from_device(b.state)
    np.testing.assert_array_equal(np.asarray(sa.loc), np.asarray(sb.loc))   # integer sums
    np.testing.assert_array_equal(np.asarray(sa.pval), np.asarray(sb.pval))
    # field value sums are fp64 per brick before the exact fixed-point total: the
    # brick shape changes their rounding (as the other blocking paths)
    np.testing.assert_allclose(np.asarray(sa.fval), np.asarray(sb.fval), rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("weights", [dict(), dict(c_f=0.5, w_d=0.3, w_p=1.5, w_f=2.0)])
def test_reuse_of_unchanged_blocks_is_exact(weights):
    """A 10-iteration run on a mid-size case where, in the later passes, many
    field blocks and point chunks reuse the previous pass's labels (unchanged
    candidates, or field bricks whose proven margin exceeds the centre moves):
    labels and centres must equal a run that recomputes everything
    (debug flag NO_REUSE), with default and with non-unit weights and time scale."""
    P = pkg()
    from paper_1903_12294_b200.engine import run_device
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
    dims, nt, ntraj = (128, 96, 64), 24, 20000
    fld, pts, _ = _synthetic(dims, nt, ntraj, 5, False, n_blobs=3)
    normalize_device(pts, fld, True)
    ext = domain_extent_device(pts, fld)
    params = P.ClusterParams(k=(8, 6, 4, 6), eps_c=1e-12, max_iterations=10, **weights)
    a = run_device(pts, fld, ext, params)
    with N.debug_options(N.DEBUG_NO_REUSE):
        b = run_device(pts, fld, ext, params)
    with N.debug_options(N.DEBUG_NO_BLOCK_CACHE):
        c = run_device(pts, fld, ext, params)
    assert torch.equal(a.field_labels, c.field_labels) and torch.equal(a.point_labels, c.point_labels)
    assert torch.equal(a.state["loc"], c.state["loc"]) and torch.equal(a.state["fval"], c.state["fval"])
    assert a.iterations_used == b.iterations_used
    assert torch.equal(a.field_labels, b.field_labels)
    assert torch.equal(a.point_labels, b.point_labels)
    sa, sb = P.CenterState.from_device(a.state), P.CenterState.from_device(b.state)
    np.testing.assert_array_equal(np.asarray(sa.loc), np.asarray(sb.loc))
    np.testing.assert_array_equal(np.asarray(sa.fval), np.asarray(sb.fval))
    np.testing.assert_array_equal(np.asarray(sa.pval), np.asarray(sb.pval))


@pytest.mark.parametrize("seed,n,n_traj,single_time,t0,presorted",
                         [(0, 5000, 300, False, 0.0, False), (1, 200000, 7000, False, 0.0, False),
                          (2, 1000, 50, True, 0.0, False), (3, 100000, 3000, False, -7.3, True),
                          (4, 50000, 400, False, 1.7e9, True), (5, 50000, 400, False, -3.0, False)])
def test_traj_split_matches_numpy(seed, n, n_traj, single_time, t0, presorted):
    """mfseg_traj_split vs the reference's lexsort + run rules (postproc.py:152-160,
    176-191): negative and sparse trajectory ids, repeated times, time gaps,
    label changes; a single unique time (stride = inf); times of both signs and
    epoch-scale times (the time keys are sorted on their varying bits only);
    records already in (trajectory, time) order (the sort is skipped)."""
    from paper_1903_12294_b200.postproc import split_trajectories_device
    rng = np.random.default_rng(seed)
    tid = rng.choice(np.arange(-50, 10 * n_traj, 10), n_traj, replace=False)[rng.integers(0, n_traj, n)]
    times = np.array([0.0]) if single_time else np.sort(rng.choice(np.arange(0, 60) * 0.25, 40,
                                                                   replace=False))
    t = times[rng.integers(0, len(times), n)] + t0
    lab = rng.integers(0, 4, n).astype(np.int32)
    if presorted:
        o = np.lexsort((t, tid))
        tid, t, lab = tid[o], t[o], lab[o]
    order, starts, stride = split_trajectories_device(torch.as_tensor(tid), torch.as_tensor(t).cuda(),
                                                      torch.as_tensor(lab))
    # numpy restatement of the reference
    u = np.unique(t)
    ref_stride = np.diff(u).min() if len(u) > 1 else np.inf
    ref_order = np.lexsort((t, tid))
    ts, ls, ids = t[ref_order], lab[ref_order], tid[ref_order]
    brk = np.ones(n, bool)
    brk[1:] = (ids[1:] != ids[:-1]) | (ls[1:] != ls[:-1]) | ((ts[1:] - ts[:-1]) > ref_stride * (1 + 1e-9))
    ref_starts = np.r_[np.flatnonzero(brk), n]
    assert stride == ref_stride
    np.testing.assert_array_equal(order.cpu().numpy(), ref_order)
    np.testing.assert_array_equal(starts.cpu().numpy(), ref_starts)


@pytest.mark.parametrize("normalize", [True, False])
def test_segment_sharded_single_rank_matches_segment(normalize):
    """parallel.segment_sharded (NCCL process group of one rank) reproduces
    pipeline.segment: same labels, centre table and NormalizationRecord."""
    import socket
    import torch.distributed as dist
    P = pkg()
    from paper_1903_12294_b200.parallel import segment_sharded
    fld, pts, tid = _synthetic((40, 32, 20), 8, 1500, 9, False)
    nt = 8
    fs = P.FieldSet((40, 32, 20), np.zeros(3), np.ones(3), np.arange(nt, dtype=float),
                    fld.values.cpu().numpy().reshape(nt, -1))
    ps = P.PointSet(tid.cpu().numpy(), pts.t.cpu().numpy(), pts.xyz.cpu().numpy(), pts.value.cpu().numpy())
    params = P.ClusterParams(k=(5, 4, 3, 2), eps_c=1e-12, max_iterations=5, normalize=normalize)
    ref, rnorm, _ = P.segment(ps, fs, params)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        seg, norm, _ = segment_sharded(ps, fs, params)
    finally:
        dist.destroy_process_group()
    assert norm == rnorm
    np.testing.assert_array_equal(seg.field_labels, ref.field_labels)
    np.testing.assert_array_equal(seg.point_labels, ref.point_labels)
    assert [c.id for c in seg.centers] == [c.id for c in ref.centers]
    np.testing.assert_array_equal([c.x_c for c in seg.centers], [c.x_c for c in ref.centers])


@pytest.mark.parametrize("flags", [0, 512])
def test_assign_crowded_vs_oracle(flags):
    """~1.4 centres per bin: candidate lists of ~100-130 exercise the 4-round
    variants of both assignment kernels and the deferral of lists > 128
    (flags 512: the deferred samples one per lane, k_deferred's path for long
    lists); labels bit-exact against the C oracle."""
    P = pkg()
    from paper_1903_12294_b200 import _native as N
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
    dims, nt, ntraj = (64, 48, 32), 12, 6000
    fld, pts, _ = _synthetic(dims, nt, ntraj, 31, False)
    normalize_device(pts, fld, True)
    ext = domain_extent_device(pts, fld)
    params = P.ClusterParams(k=(5, 4, 3, 3), w_d=0.6)
    rng = np.random.default_rng(31)
    C = P.interval_distances(ext, params.k)
    seeds = P.seed_centers(ext, params.k)
    extra = seeds[rng.integers(0, len(seeds), int(0.45 * len(seeds)))]
    loc = np.vstack([seeds, extra]) + rng.uniform(-0.4, 0.4, (len(seeds) + len(extra), 4)) * C
    K = len(loc)
    cs = P.CenterState.from_seeds(loc)
    cs.pval = np.where(rng.random(K) < 0.8, rng.random(K), np.nan)
    cs.fval = np.where(rng.random(K) < 0.8, rng.random(K), np.nan)
    cs.has_p, cs.has_f = ~np.isnan(cs.pval), ~np.isnan(cs.fval)
    grid = P.CenterGrid(cs.loc, ext, C, params.k)
    fs = P.FieldSet(dims, np.zeros(3), np.ones(3), fld.times.cpu().numpy(),
                    fld.values.cpu().numpy().reshape(nt, -1))
    ps = P.PointSet(np.zeros(pts.n, np.int64), pts.t.cpu().numpy(), pts.xyz.cpu().numpy(),
                    pts.value.cpu().numpy())
    with N.debug_options(flags):
        pl, fl = P.assign_iteration(ps, fs, None, cs, grid, params, C)
    want_p, want_f = _oracle_labels(ps, fs, cs, ext, C, params)
    np.testing.assert_array_equal(fl, want_f)
    np.testing.assert_array_equal(pl, want_p)


@pytest.mark.parametrize("n_slots,nt,ncell", [(7, 3, 10000), (256, 2, 70001), (300, 4, 5000),
                                              (1, 1, 4097), (49, 5, 4096 * 3)])
def test_voxel_csr_paths_vs_numpy(n_slots, nt, ncell):
    """mfseg_voxel_csr (counting sort for <= 256 features, radix sort above):
    per (timestep, feature) ascending cell lists equal the reference's
    flatnonzero(lab_m == fid) (postproc.py:162-168)."""
    from paper_1903_12294_b200.postproc import voxel_csr_device
    rng = np.random.default_rng(n_slots + nt)
    # spatially coherent labels with noise, like real segmentations
    lab = (np.arange(nt * ncell) // 997 + rng.integers(0, 3, nt * ncell)) % n_slots
    lab = lab.astype(np.int32)
    seg, cells = voxel_csr_device(torch.as_tensor(lab).cuda(), nt, ncell, n_slots)
    seg, cells = seg.cpu().numpy(), cells.cpu().numpy()
    for m in range(nt):
        lm = lab[m * ncell:(m + 1) * ncell]
        for s in range(n_slots):
            want = np.flatnonzero(lm == s)
            a, b = seg[m * n_slots + s], seg[m * n_slots + s + 1]
            np.testing.assert_array_equal(cells[a:b], want)
    assert seg[-1] == nt * ncell


@pytest.mark.parametrize("n_slots", [3, 320, 321, 2000])
def test_feature_stats_smem_and_global_paths_agree(n_slots):
    """k_stats accumulates in shared memory for <= 320 features and with global
    atomics above; both must equal a numpy restatement of feature_stats
    (postproc.py:194-227) on random slots (exact bbox / counts, mean / std 1e-12)."""
    from paper_1903_12294_b200.engine import DeviceField, DevicePoints
    from paper_1903_12294_b200.postproc import feature_stats_device
    rng = np.random.default_rng(n_slots)
    dims, nt, npnt = (17, 9, 6), 3, 5000
    ncell = int(np.prod(dims))
    fv = rng.random(nt * ncell)
    fld = DeviceField(dims, np.array([0.5, -1.0, 2.0]), np.array([0.25, 1.5, 1.0]),
                      torch.tensor([0.0, 1.0, 2.5], dtype=torch.float64, device="cuda"),
                      torch.as_tensor(fv).cuda())
    xyz, t, pv = rng.random((npnt, 3)) * 5, rng.random(npnt) * 3, rng.random(npnt)
    pts = DevicePoints(torch.as_tensor(xyz).cuda(), torch.as_tensor(t).cuda(), torch.as_tensor(pv).cuda())
    fs = rng.integers(-1, n_slots, nt * ncell).astype(np.int32)
    ps = rng.integers(-1, n_slots, npnt).astype(np.int32)
    rows = feature_stats_device(n_slots, fld, torch.as_tensor(fs).cuda(), pts, torch.as_tensor(ps).cuda())
    ii, jj, kk = np.meshgrid(np.arange(dims[0]), np.arange(dims[1]), np.arange(dims[2]), indexing="ij")
    cx = 0.5 + (ii.transpose(2, 1, 0).ravel() + 0.5) * 0.25
    cy = -1.0 + (jj.transpose(2, 1, 0).ravel() + 0.5) * 1.5
    cz = 2.0 + (kk.transpose(2, 1, 0).ravel() + 0.5) * 1.0
    floc = np.column_stack([np.tile(cx, nt), np.tile(cy, nt), np.tile(cz, nt),
                            np.repeat([0.0, 1.0, 2.5], ncell)])
    ploc = np.column_stack([xyz, t])
    for s in range(0, n_slots, max(1, n_slots // 17)):
        f, p = fs == s, ps == s
        loc = np.vstack([floc[f], ploc[p]])
        if len(loc) == 0:
            continue
        np.testing.assert_array_equal(rows[s][0:4], loc.min(0))
        np.testing.assert_array_equal(rows[s][4:8], loc.max(0))
        assert rows[s][12] == p.sum() and rows[s][13] == f.sum()
        if p.any():
            assert abs(rows[s][8] - pv[p].mean()) <= 1e-12 and abs(rows[s][9] - pv[p].std()) <= 1e-12
        if f.any():
            assert abs(rows[s][10] - fv[f].mean()) <= 1e-12 and abs(rows[s][11] - fv[f].std()) <= 1e-12


@pytest.mark.parametrize("seed,n,eps", [(0, 3000, 0.05), (1, 2500, 0.3), (2, 400, 1e-3)])
def test_merge_random_tables_vs_oracle(seed, n, eps):
    """mfseg_merge (p_c-sorted window sweep, cached-parent union-find, lane-split
    ordered sums) against the oracle's all-pairs restatement of postproc.py:59-92
    on random tables: absent values (None), both signs, values near DELTA,
    duplicates and clusters of near-equal values; merge map and merged rows
    bit-identical."""
    P = pkg()
    from oracle import mfseg_oracle as O
    rng = np.random.default_rng(seed)
    base = rng.choice([0.1, 0.5, 2.0, -0.7, 3e-13], n)
    pc = base * (1 + rng.normal(0, eps / 3, n))
    fc = rng.choice([1.0, -4.0, 0.25], n) * (1 + rng.normal(0, eps / 3, n))
    pc[rng.random(n) < 0.1] = np.nan
    fc[rng.random(n) < 0.1] = np.nan
    pc[: n // 50] = pc[n // 50: 2 * (n // 50)]           # exact duplicates
    ids = np.sort(rng.choice(10 * n, n, replace=False))
    n_p = np.where(np.isnan(pc), 0, rng.integers(1, 50, n))
    n_f = np.where(np.isnan(fc), 0, rng.integers(1, 500, n))
    n_f[(n_p == 0) & (n_f == 0)] = 1
    fc[(n_f > 0) & np.isnan(fc)] = 0.5
    loc = rng.random((n, 4)) * 100 - 20
    rows = [P.ClusterCenter(int(i), *map(float, l), None if np.isnan(p) else float(p),
                            None if np.isnan(f) else float(f), int(a), int(b))
            for i, l, p, f, a, b in zip(ids, loc, pc, fc, n_p, n_f)]
    orows = [O.Summary(int(i), l.copy(), None if np.isnan(p) else float(p), None if np.isnan(f) else float(f),
                       int(a), int(b)) for i, l, p, f, a, b in zip(ids, loc, pc, fc, n_p, n_f)]
    mm, merged = P.merge_clusters(rows, eps)
    omm, omerged = O.merge(orows, eps)
    assert mm == omm
    assert len(merged) == len(omerged) and len(merged) < n
    for g, o in zip(merged, omerged):
        assert g.id == o.id and g.n_points == o.n_points and g.n_fields == o.n_fields
        assert (g.x_c, g.y_c, g.z_c, g.t_c) == tuple(float(v) for v in o.loc)
        assert g.p_c == o.p_c and g.f_c == o.f_c
