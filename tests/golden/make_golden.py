"""Generate golden vectors for the segmentation hot path FROM THE REFERENCE ITSELF.

This script is test infrastructure. It imports the unmodified reference package
(`mfseg`, /root/reference/pkg/src) in the build container, runs it on small
seeded inputs and writes the inputs together with the reference's outputs as
compressed fixtures next to this file.  The GPU box has no /root/reference, so
the committed fixtures are what `tests/` compares against there.

Run:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Cases (reference call sites in brackets):
  * run_*      full `pipeline.segment` / `engine.run` results         [engine.py:323-381]
  * assign_*   one `engine.assign_iteration` with given centers        [engine.py:208-241]
  * accum_*    `engine.accumulate` + `update_centers` on given labels  [engine.py:244-286]
  * merge/features for run cases                                       [postproc.py:59-227]
  * link_*     `ingest.build_link_index`                               [ingest.py:261-280]
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import mfseg  # noqa: F401
    from mfseg import engine, ingest, pipeline, postproc  # noqa: F401
    return mfseg


mf = _import_reference()
from mfseg import engine, ingest, pipeline, postproc  # noqa: E402
from mfseg.ingest import Blob, SyntheticSpec  # noqa: E402
from mfseg.model import ClusterParams, DomainExtent, FieldSet, PointSet  # noqa: E402

UNIT = DomainExtent(0, 10, 0, 10, 0, 10, 0, 4)


# ---------------------------------------------------------------- dataset specs
# These mirror the shapes of the reference's own fixtures (tests/conftest.py)
# so the goldens exercise the same regimes the reference tests do.

def spec_slabs(n_blobs, seed=11, noise=0.0, traj=20, bg_traj=20):
    n = n_blobs + 1
    w = 10.0 / n
    blobs, lab = [], 1
    for s in range(n):
        if s == n // 2:
            continue
        blobs.append(Blob(label=lab, shape="box", center=((s + 0.5) * w, 5, 5),
                          radii=(w / 2, 5, 5), t_start=0, t_end=4,
                          field_value=float(lab), point_value=float(lab),
                          n_trajectories=traj))
        lab += 1
    return SyntheticSpec(extent=UNIT, grid_dims=(3 * n, 6, 6), n_field_steps=5,
                         n_point_steps=10, blobs=tuple(blobs), n_background_trajectories=bg_traj,
                         field_noise=noise, point_noise=noise, seed=seed)


def spec_two_blob(seed=7, noise=0.0):
    return SyntheticSpec(
        extent=UNIT, grid_dims=(12, 8, 8), n_field_steps=5, n_point_steps=10,
        blobs=(Blob(label=1, center=(2.2, 5, 5), radii=(1.4, 1.4, 1.4), t_start=0, t_end=4,
                    field_value=1.0, point_value=1.0, n_trajectories=25),
               Blob(label=2, center=(7.8, 5, 5), radii=(1.4, 1.4, 1.4), t_start=0, t_end=4,
                    field_value=2.0, point_value=2.0, n_trajectories=25)),
        n_background_trajectories=20, field_noise=noise, point_noise=noise, seed=seed)


def spec_blob_field(n_samples, noise=0.0, velocity=0.0, seed=3):
    steps, nx = 8, 40
    nz = max(int(round(n_samples * 0.8 / (steps * nx * nx))), 1)
    ntraj = max((n_samples - nx * nx * nz * steps) // steps, 100)
    blobs = tuple(Blob(label=i + 1, center=(2.5 + 1.5 * i, 2.5 + 1.5 * i, 5.0),
                       radii=(1.2, 1.2, 1.2), t_start=0, t_end=4,
                       velocity=(velocity, velocity * 0.4, 0),
                       field_value=1.0 + i, point_value=2.0 + i,
                       n_trajectories=ntraj // 4) for i in range(3))
    return SyntheticSpec(extent=UNIT, grid_dims=(nx, nx, nz), n_field_steps=steps,
                         n_point_steps=steps, blobs=blobs,
                         n_background_trajectories=ntraj - 3 * (ntraj // 4),
                         field_noise=noise, point_noise=noise, seed=seed)


# ---------------------------------------------------------------- serialisers

def pack_points(prefix, ps):
    return {f"{prefix}traj_id": ps.traj_id.astype(np.int64), f"{prefix}t": ps.t,
            f"{prefix}xyz": ps.xyz, f"{prefix}value": ps.value}


def pack_field(prefix, fs):
    return {f"{prefix}dims": np.asarray(fs.dims, np.int64), f"{prefix}origin": fs.origin,
            f"{prefix}spacing": fs.spacing, f"{prefix}times": fs.times,
            f"{prefix}values": fs.values}


def pack_centers(prefix, centers):
    f = lambda v: np.nan if v is None else v  # noqa: E731
    return {
        f"{prefix}id": np.array([c.id for c in centers], np.int64),
        f"{prefix}loc": np.array([[c.x_c, c.y_c, c.z_c, c.t_c] for c in centers]).reshape(-1, 4),
        f"{prefix}p_c": np.array([f(c.p_c) for c in centers], float),
        f"{prefix}f_c": np.array([f(c.f_c) for c in centers], float),
        f"{prefix}n_points": np.array([c.n_points for c in centers], np.int64),
        f"{prefix}n_fields": np.array([c.n_fields for c in centers], np.int64),
    }


def pack_state(prefix, cs):
    return {f"{prefix}loc": cs.loc, f"{prefix}pval": cs.pval, f"{prefix}fval": cs.fval,
            f"{prefix}has_p": cs.has_p, f"{prefix}has_f": cs.has_f,
            f"{prefix}n_points": cs.n_points, f"{prefix}n_fields": cs.n_fields,
            f"{prefix}dormant": cs.dormant}


def features_doc(feats):
    out = []
    for f in feats:
        s = f.stats
        out.append({
            "id": int(f.id), "member_clusters": [int(m) for m in f.member_clusters],
            "polylines": [[int(i) for i in line] for line in f.polylines],
            "isolated_points": [int(i) for i in f.isolated_points],
            "voxels": {str(m): [int(i) for i in cells] for m, cells in sorted(f.voxels.items())},
            "stats": s.to_dict() if s else None,
        })
    return out


def save(name, arrays, meta):
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print(f"wrote {name}: {sum(a.nbytes for a in arrays.values())} raw bytes")


# ---------------------------------------------------------------- cases

def run_case(name, points, fields, params, normalize_here, merge_eps=(), extent=None,
             with_features=True):
    """Full segmentation through the reference, plus merge + features."""
    deltas = []
    if normalize_here:
        seg, norm, _ = pipeline.segment(points, fields, params,
                                        progress=lambda it, d: deltas.append((it, d)))
        p_n, f_n, _ = ingest.normalize_variables(points, fields, params.normalize)
        ext = ingest.domain_extent(p_n, f_n)
        norm_d = norm.to_dict()
    else:
        p_n, f_n, ext, norm_d = points, fields, extent, None
        seg = engine.run(points, fields, extent, params,
                         progress=lambda it, d: deltas.append((it, d)))
    p_n = p_n if p_n is not None else PointSet.empty()
    f_n = f_n if f_n is not None else FieldSet.empty()
    arrays = {}
    arrays.update(pack_points("in_p_", p_n))
    arrays.update(pack_field("in_f_", f_n))
    if normalize_here:   # raw values, to check min-max normalization (ingest.py:312-335)
        arrays["in_raw_p_value"] = points.value if points is not None else np.zeros(0)
        arrays["in_raw_f_values"] = fields.values if fields is not None else np.zeros((0, 1))
    arrays["out_point_labels"] = seg.point_labels.astype(np.int32)
    arrays["out_field_labels"] = seg.field_labels.astype(np.int32)
    arrays.update(pack_centers("out_c_", seg.centers))
    meta = {"params": params.to_dict(), "extent": ext.to_dict(), "normalization": norm_d,
            "iterations_used": seg.iterations_used, "converged": bool(seg.converged),
            "progress": [[int(i), float(d)] for i, d in deltas], "merges": {},
            "source": "reference mfseg 0.1.0 (/root/reference/pkg/src), " + name}
    for eps in merge_eps:
        mm, merged = postproc.merge_clusters(seg.centers, eps)
        key = repr(float(eps))
        ids = np.array(sorted(mm), np.int64)
        arrays[f"merge_{key}_ids"] = ids
        arrays[f"merge_{key}_rep"] = np.array([mm[i] for i in ids], np.int64)
        arrays.update(pack_centers(f"merge_{key}_c_", merged))
        meta["merges"][key] = len(merged)
        if with_features:
            feats = postproc.build_features(seg, mm, p_n, f_n)
            meta.setdefault("features", {})[key] = features_doc(feats)
    if with_features:
        feats = postproc.build_features(seg, None, p_n, f_n)
        meta.setdefault("features", {})["identity"] = features_doc(feats)
    save(name, arrays, meta)


def load_via_files(spec):
    """Same flow as the frontend fixtures: write_synthetic -> load_dataset."""
    with tempfile.TemporaryDirectory() as d:
        paths = ingest.write_synthetic(d, spec)
        points, fields = pipeline.load_dataset(paths["field"], paths["points"], "v")
    return points, fields


def assign_case(name, points, fields, extent, params, cs, note):
    C = engine.interval_distances(extent, params.k)
    grid = engine.CenterGrid(cs.loc, extent, C, params.k)
    floc = fields.loc4() if len(fields) else np.empty((0, 4))
    pl, fl = engine.assign_iteration(points, fields, floc, cs, grid, params, C)
    sums = engine.accumulate(pl, points, fl, fields, floc, len(cs.loc))
    new = engine.update_centers(cs, *sums)
    arrays = {}
    arrays.update(pack_points("in_p_", points))
    arrays.update(pack_field("in_f_", fields))
    arrays.update(pack_state("in_c_", cs))
    arrays["out_point_labels"] = pl.astype(np.int64)
    arrays["out_field_labels"] = fl.astype(np.int64)
    for nm, a in zip(("sums", "psum", "fsum", "n_p", "n_f"), sums):
        arrays[f"out_acc_{nm}"] = a
    arrays.update(pack_state("out_new_", new))
    meta = {"params": params.to_dict(), "extent": extent.to_dict(), "note": note,
            "converged": bool(engine.has_converged(cs, new, params.eps_c)),
            "max_delta": float(engine.max_center_delta(cs, new)),
            "source": "reference mfseg 0.1.0 engine.assign_iteration/accumulate/update_centers"}
    save(name, arrays, meta)


def make_points(loc, values):
    loc = np.asarray(loc, float)
    return PointSet(np.arange(len(loc)), loc[:, 3].copy(), loc[:, :3].copy(),
                    np.asarray(values, float))


FRONTEND = "/root/reference/pkg/frontend/test/fixtures"


def frontend_subset():
    """Numeric subset of the reference's recorded service responses (the only
    end-to-end golden vectors the reference ships), stored alongside our case."""
    def rd(n):
        with open(os.path.join(FRONTEND, n)) as fh:
            return json.load(fh)
    keys = ("id", "x_c", "y_c", "z_c", "t_c", "p_c", "f_c", "n_points", "n_fields",
            "bbox_min", "bbox_max", "p_std", "f_std")
    return {
        "centers_all": [{k: c[k] for k in keys} for c in rd("centers_all.json")["centers"]],
        "centers_merged_eps2": [{k: c[k] for k in keys} for c in rd("centers_merged.json")["centers"]],
        "merge_all": rd("merge_all.json"),
        "feature0_stats": rd("feature_full.json")["stats"],
    }


def artifacts_case():
    """The reference's own artifact writer (artifacts.py) on the frontend
    configuration: segmentation.json + label files, merge.json, features.json
    -> tests/golden/artifacts_slab2/ (byte-level goldens for our writer)."""
    from mfseg import artifacts
    out = os.path.join(HERE, "artifacts_slab2")
    os.makedirs(out, exist_ok=True)
    pts, fld = load_via_files(spec_slabs(2))
    params = ClusterParams(k=(3, 1, 1, 1), w_d=0.05, eps_m=0.01, normalize=True)
    seg, norm, _ = pipeline.segment(pts, fld, params)
    artifacts.save_segmentation(out, seg, norm)
    mm, merged = postproc.merge_clusters(seg.centers, 0.01)
    artifacts.save_merge(out, 0.01, mm, merged)
    p_n, f_n, _ = ingest.normalize_variables(pts, fld, True)
    feats = postproc.build_features(seg, mm, p_n, f_n)
    artifacts.save_features(out, feats, merged, mm)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "artifacts":
        artifacts_case()
        return
    # 1. the frontend golden configuration (pkg/frontend/test/fixtures/*):
    #    slab_spec(2), k=(3,1,1,1), w_d=0.05, eps_m=0.01, normalize on
    pts, fld = load_via_files(spec_slabs(2))
    run_case("run_slab2_frontend", pts, fld,
             ClusterParams(k=(3, 1, 1, 1), w_d=0.05, eps_m=0.01, normalize=True),
             normalize_here=True, merge_eps=(0.01, 2.0))
    with open(os.path.join(HERE, "run_slab2_frontend.json")) as fh:
        meta = json.load(fh)
    meta["frontend_fixture"] = frontend_subset()
    with open(os.path.join(HERE, "run_slab2_frontend.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
        fh.write("\n")

    # 2. two-blob dataset, k=(2,2,2,2), w_d=0.2 (test_engine determinism case)
    fs, ps, _, _ = ingest.generate_synthetic(spec_two_blob())
    run_case("run_two_blob", ps, fs, ClusterParams(k=(2, 2, 2, 2), w_d=0.2),
             normalize_here=True, merge_eps=(0.01,))

    # 3. noisy drifting blobs, 2e4 samples, k=(3,3,2,2), w_d=0.5 (determinism acceptance)
    fs, ps, _, _ = ingest.generate_synthetic(spec_blob_field(20000, noise=0.05, velocity=0.3))
    run_case("run_blob_noisy", ps, fs, ClusterParams(k=(3, 3, 2, 2), w_d=0.5),
             normalize_here=True, merge_eps=(0.01, 0.1))

    # 4. larger continuous case, more clusters, the survey's timing protocol
    fs, ps, _, _ = ingest.generate_synthetic(spec_blob_field(60000, noise=0.05, velocity=0.5,
                                                             seed=9))
    run_case("run_blob_k256", ps, fs,
             ClusterParams(k=(4, 4, 4, 4), w_d=1.0, eps_c=1e-12, max_iterations=10),
             normalize_here=True, merge_eps=(0.05,), with_features=False)

    # 5. field-only and point-only runs (unnormalized, fixed extent)
    fs, ps, _, _ = ingest.generate_synthetic(spec_two_blob())
    run_case("run_field_only", None, fs, ClusterParams(k=(2, 1, 1, 1), normalize=False),
             normalize_here=False, extent=UNIT, merge_eps=(0.01,))
    run_case("run_point_only", ps, None, ClusterParams(k=(2, 1, 1, 1), normalize=False),
             normalize_here=False, extent=UNIT, merge_eps=(0.01,))

    # 6. background merge acceptance configuration (test_acceptance.py:198-226)
    blob = Blob(label=1, shape="box", center=(9.75, 5, 5), radii=(0.25, 4, 4), t_start=0,
                t_end=4, field_value=0.0, point_value=5.0, n_trajectories=15)
    spec = SyntheticSpec(extent=UNIT, grid_dims=(40, 6, 6), n_field_steps=5, n_point_steps=10,
                         blobs=(blob,), n_background_trajectories=80, seed=2)
    fs, ps, _, _ = ingest.generate_synthetic(spec)
    run_case("run_background_merge", ps, fs, ClusterParams(k=(20, 1, 1, 1), normalize=False),
             normalize_here=False, extent=UNIT, merge_eps=(0.01,))

    # 7. striped field, weight trade-off (test_acceptance.py:165-194), both weights
    ext = DomainExtent(0, 8, 0, 4, 0, 1, 0, 1)
    nx, ny, nz = 32, 16, 2
    xs = (np.arange(nx) + 0.5) * 8 / nx
    vals = np.tile((np.floor(xs / 0.9) % 2).astype(float), ny * nz)
    fs = FieldSet((nx, ny, nz), np.zeros(3), np.array([8 / nx, 4 / ny, 1 / nz]),
                  np.array([0.0, 1.0]), np.vstack([vals, vals]))
    for tag, wd in (("lo", 0.01), ("hi", 10.0)):
        run_case(f"run_stripes_{tag}", None, fs,
                 ClusterParams(k=(4, 2, 1, 1), w_d=wd, w_f=1.0, normalize=False,
                               max_iterations=30),
                 normalize_here=False, extent=ext, with_features=False)

    # ---- step-level assignment cases (given centers) ----
    # 8. oracle-equivalence instance (test_acceptance.py:33-75)
    params = ClusterParams(k=(4, 4, 4, 4), w_d=1.0, w_p=0.1, w_f=0.1)
    rng = np.random.default_rng(21)
    loc = rng.random((6000, 4)) * [10, 10, 10, 4]
    ps = PointSet(np.arange(6000), loc[:, 3], loc[:, :3].copy(), rng.random(6000))
    fs = FieldSet((10, 10, 10), np.zeros(3), np.ones(3), np.linspace(0, 4, 4),
                  rng.random((4, 1000)))
    C = engine.interval_distances(UNIT, params.k)
    K = params.k_total
    cs = engine.CenterState.from_seeds(engine.seed_centers(UNIT, params.k)
                                       + rng.uniform(-1, 1, (K, 4)) * C / 32)
    cs.pval, cs.fval = rng.random(K), rng.random(K)
    cs.has_p, cs.has_f = np.ones(K, bool), np.ones(K, bool)
    assign_case("assign_oracle_equiv", ps, fs, UNIT, params, cs,
                "test_acceptance.py:33-75 instance")

    # 9. stranded sample (test_engine.py:136-148)
    ext = DomainExtent(0, 16, 0, 1, 0, 1, 0, 1)
    params = ClusterParams(k=(8, 1, 1, 1), w_d=1.0, w_p=1.0)
    cs = engine.CenterState.from_seeds(np.array([[1.0, 0.5, 0.5, 0.5], [3.0, 0.5, 0.5, 0.5]]))
    cs.pval = np.array([0.9, 0.1])
    cs.has_p = np.array([True, True])
    assign_case("assign_stranded", make_points([[15.0, 0.5, 0.5, 0.5]], [0.1]),
                FieldSet.empty(), ext, params, cs, "test_engine.py:136-148")

    # 10. hard random instances: strong drift (stranded + crowded bins), absent
    #     values, dormant centers, exact-boundary samples and exact ties.
    for seed in range(4):
        rng = np.random.default_rng(100 + seed)
        k = [(3, 4, 2, 3), (5, 2, 3, 2), (2, 2, 2, 2), (6, 5, 1, 4)][seed]
        ext = DomainExtent(-2.0, 6.0, 0.0, 3.0, 1.0, 2.5, 0.0, 7.0)
        params = ClusterParams(k=k, c_f=[1.0, 0.5, 2.0, 1.25][seed], w_d=[1.0, 0.3, 2.0, 0.05][seed],
                               w_p=[1.0, 0.0, 0.7, 2.0][seed], w_f=[0.5, 1.5, 0.0, 1.0][seed])
        K = int(np.prod(k))
        Cd = engine.interval_distances(ext, k)
        seeds = engine.seed_centers(ext, k)
        drift = [0.3, 1.5, 0.8, 2.5][seed]
        cs = engine.CenterState.from_seeds(seeds + rng.uniform(-drift, drift, (K, 4)) * Cd)
        # pile a few centers onto one bin (crowding)
        cs.loc[: max(K // 6, 2)] = cs.loc[0] + rng.uniform(-0.1, 0.1, (max(K // 6, 2), 4)) * Cd
        cs.pval = np.where(rng.random(K) < 0.8, rng.random(K), np.nan)
        cs.fval = np.where(rng.random(K) < 0.8, rng.random(K), np.nan)
        cs.has_p, cs.has_f = ~np.isnan(cs.pval), ~np.isnan(cs.fval)
        cs.dormant = rng.random(K) < 0.1
        nx, ny, nz, nt = [(9, 5, 4, 6), (16, 3, 2, 5), (7, 7, 3, 3), (12, 6, 1, 8)][seed]
        sp = np.array([8.0 / nx, 3.0 / ny, 1.5 / nz])
        times = np.sort(rng.choice(np.linspace(0, 7, 29), nt, replace=False))
        if seed == 2:
            fvals = np.round(rng.random((nt, nx * ny * nz)) * 4) / 4   # many exact ties
        else:
            fvals = rng.random((nt, nx * ny * nz))
        fs = FieldSet((nx, ny, nz), np.array([-2.0, 0.0, 1.0]), sp, times, fvals)
        n = 3000
        loc = rng.random((n, 4)) * (ext.maxs - ext.mins) + ext.mins
        # exact bin-boundary and box-boundary coordinates
        loc[:300] = np.round(loc[:300] / (Cd / 2)) * (Cd / 2)
        loc[:300] = np.clip(loc[:300], ext.mins, ext.maxs)
        pv = rng.random(n)
        pv[:200] = np.round(pv[:200] * 2) / 2
        assign_case(f"assign_hard_{seed}", make_points(loc, pv), fs, ext, params, cs,
                    f"random hard instance seed {seed}")

    # 11. initial assignment on a regular lattice: exact ties everywhere
    params = ClusterParams(k=(2, 2, 2, 2), c_f=1.0)
    ext = DomainExtent(0, 4, 0, 4, 0, 4, 0, 4)
    g = np.arange(0, 4.01, 0.5)
    loc = np.array(np.meshgrid(g, g, g, g, indexing="ij")).reshape(4, -1).T
    cs = engine.CenterState.from_seeds(engine.seed_centers(ext, params.k))
    zero = ClusterParams(k=params.k, w_d=1.0, w_p=0.0, w_f=0.0)
    fs = FieldSet((4, 4, 4), np.zeros(3), np.ones(3), np.array([0.0, 1.0, 2.0, 3.0, 4.0]),
                  np.zeros((5, 64)))
    assign_case("assign_lattice_ties", make_points(loc, np.zeros(len(loc))), fs, ext, zero, cs,
                "initial-pass lattice with exact equidistant ties")

    # ---- link index (ingest.py:261-280) ----
    fs, ps, _, _ = ingest.generate_synthetic(spec_blob_field(20000, noise=0.05, velocity=0.3))
    kept, dropped = ingest.filter_to_grid(ps, fs)
    li = ingest.build_link_index(fs, kept)
    keys = list(li.buckets)   # insertion order = the reference's flat-key order
    arrays = pack_points("in_p_", kept)
    arrays.update(pack_field("in_f_", fs))
    arrays["out_keys"] = np.array(keys, np.int64).reshape(-1, 4)
    arrays["out_sizes"] = np.array([len(li.buckets[k]) for k in keys], np.int64)
    arrays["out_members"] = (np.concatenate([li.buckets[k] for k in keys]).astype(np.int64)
                             if keys else np.zeros(0, np.int64))
    save("link_blob", arrays, {"dropped": dropped, "source": "reference ingest.build_link_index"})


if __name__ == "__main__":
    main()
