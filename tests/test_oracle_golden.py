"""Pin the CPU oracle (numpy + C restatements) to the reference's own outputs.

The golden vectors were produced by running the reference package itself
(tests/golden/make_golden.py).  Everything here is exact-equality unless the
reference's own value is only defined up to summation order.
"""
import numpy as np
import pytest

from golden_io import Case, names
from oracle import c_oracle
from oracle import mfseg_oracle as O

RUNS = names("run_")
ASSIGNS = names("assign_")


def _table_arrays(cs):
    ids = cs.live_ids()
    return ids, cs.loc[ids], np.where(cs.has_p[ids], cs.pval[ids], np.nan), \
        np.where(cs.has_f[ids], cs.fval[ids], np.nan)


def _oracle_run(case, impl):
    p = case.params
    dims, origin, spacing, times, values = case.field
    mins, maxs = case.extent
    kw = dict(c_f=p["c_f"], w_d=p["w_d"], w_p=p["w_p"], w_f=p["w_f"], eps_c=p["eps_c"],
              max_iterations=p["max_iterations"])
    if impl == "numpy":
        r = O.segment(case.p_loc, case["in_p_value"], dims, origin, spacing, times, values,
                      mins, maxs, p["k"], **kw)
        ids, loc, pc, fc = _table_arrays(r.centres)
        return (r.point_labels, r.field_labels, ids, loc, pc, fc, r.iterations_used,
                r.converged, [d for _, d in r.progress])
    if impl == "c_grid":
        r = c_oracle.run_grid(case.p_loc, case["in_p_value"], dims, origin, spacing, times,
                              values.reshape(-1), mins, maxs, p["k"], threads=4, **kw)
    else:
        floc = O.field_locations(dims, origin, spacing, times) if values.size else np.zeros((0, 4))
        r = c_oracle.run(case.p_loc, case["in_p_value"], floc, values.reshape(-1), mins, maxs,
                         p["k"], threads=4, **kw)
    ids = np.flatnonzero(r["n_points"] + r["n_fields"] > 0)
    pc = np.where(r["has_p"][ids], r["pval"][ids], np.nan)
    fc = np.where(r["has_f"][ids], r["fval"][ids], np.nan)
    return (r["point_labels"], r["field_labels"], ids, r["loc"][ids], pc, fc,
            r["iterations_used"], r["converged"], list(r["progress"]))


@pytest.mark.parametrize("impl", ["numpy", "c", "c_grid"])
@pytest.mark.parametrize("name", RUNS)
def test_run_matches_reference_bit_exact(name, impl):
    case = Case(name)
    pl, fl, ids, loc, pc, fc, it, conv, prog = _oracle_run(case, impl)
    np.testing.assert_array_equal(pl, case["out_point_labels"])
    np.testing.assert_array_equal(fl, case["out_field_labels"])
    np.testing.assert_array_equal(ids, case["out_c_id"])
    np.testing.assert_array_equal(loc, case["out_c_loc"])      # same sequential sums
    np.testing.assert_array_equal(pc, case["out_c_p_c"])
    np.testing.assert_array_equal(fc, case["out_c_f_c"])
    assert it == case.meta["iterations_used"] and conv == case.meta["converged"]
    np.testing.assert_array_equal(prog, [d for _, d in case.meta["progress"]])


@pytest.mark.parametrize("name", ASSIGNS)
def test_assign_matches_reference(name):
    case = Case(name)
    p = case.params
    mins, maxs = case.extent
    C = O.interval_lengths(mins, maxs, p["k"])
    cloc = case["in_c_loc"]
    tab = O.NeighbourTable(cloc, mins, C, p["k"])
    pl = O.assign_kind(case.p_loc, case["in_p_value"], cloc, case["in_c_pval"], case["in_c_has_p"],
                       tab, p["w_p"], p["w_d"], p["c_f"], C)
    dims, origin, spacing, times, values = case.field
    floc = O.field_locations(dims, origin, spacing, times) if values.size else np.zeros((0, 4))
    fl = O.assign_kind(floc, values.reshape(-1), cloc, case["in_c_fval"], case["in_c_has_f"],
                       tab, p["w_f"], p["w_d"], p["c_f"], C)
    np.testing.assert_array_equal(pl, case["out_point_labels"])
    np.testing.assert_array_equal(fl, case["out_field_labels"])
    # C restatement, same inputs
    cpl = c_oracle.assign(case.p_loc, case["in_p_value"], cloc, case["in_c_pval"],
                          case["in_c_has_p"], mins, C, p["k"], p["w_p"], p["w_d"], p["c_f"])
    cfl = c_oracle.assign(floc, values.reshape(-1), cloc, case["in_c_fval"], case["in_c_has_f"],
                          mins, C, p["k"], p["w_f"], p["w_d"], p["c_f"])
    np.testing.assert_array_equal(cpl, case["out_point_labels"])
    np.testing.assert_array_equal(cfl, case["out_field_labels"])
    if values.size:   # field cells from the geometry, all and a shuffled subset
        gfl = c_oracle.assign_field(dims, origin, spacing, times, values, cloc, case["in_c_fval"],
                                    case["in_c_has_f"], mins, C, p["k"], p["w_f"], p["w_d"],
                                    p["c_f"])
        np.testing.assert_array_equal(gfl, case["out_field_labels"])
        idx = np.random.default_rng(0).permutation(values.size)[: max(values.size // 3, 1)]
        sfl = c_oracle.assign_field(dims, origin, spacing, times, values, cloc, case["in_c_fval"],
                                    case["in_c_has_f"], mins, C, p["k"], p["w_f"], p["w_d"],
                                    p["c_f"], idx=idx)
        np.testing.assert_array_equal(sfl, case["out_field_labels"][idx])
    # accumulate + update with the reference's labels
    K = len(cloc)
    sums = O.cluster_sums(case["out_point_labels"], case.p_loc, case["in_p_value"],
                          case["out_field_labels"], floc, values.reshape(-1), K)
    for nm, got in zip(("sums", "psum", "fsum", "n_p", "n_f"), sums):
        np.testing.assert_array_equal(got, case[f"out_acc_{nm}"])
    old = O.Centres(cloc, case["in_c_pval"], case["in_c_fval"], case["in_c_has_p"],
                    case["in_c_has_f"], case["in_c_n_points"], case["in_c_n_fields"],
                    case["in_c_dormant"])
    new = O.refresh_centres(old, *sums)
    for f in ("loc", "pval", "fval", "has_p", "has_f", "n_points", "n_fields", "dormant"):
        np.testing.assert_array_equal(getattr(new, f), case[f"out_new_{f}"])
    assert O.is_converged(old, new, p["eps_c"]) == case.meta["converged"]
    assert O.largest_change(old, new) == case.meta["max_delta"]


def _rows_from(case, prefix):
    out = []
    for i, loc, pc, fc, n_p, n_f in zip(case[prefix + "id"], case[prefix + "loc"],
                                        case[prefix + "p_c"], case[prefix + "f_c"],
                                        case[prefix + "n_points"], case[prefix + "n_fields"]):
        out.append(O.Summary(int(i), np.asarray(loc), None if np.isnan(pc) else float(pc),
                             None if np.isnan(fc) else float(fc), int(n_p), int(n_f)))
    return out


@pytest.mark.parametrize("name", RUNS)
def test_merge_and_features_match_reference(name):
    case = Case(name)
    rows = _rows_from(case, "out_c_")
    dims, origin, spacing, times, values = case.field
    for key in case.meta["merges"]:
        mm, merged = O.merge(rows, float(key))
        ids = case[f"merge_{key}_ids"]
        assert [mm[int(i)] for i in ids] == list(case[f"merge_{key}_rep"])
        want = _rows_from(case, f"merge_{key}_c_")
        assert [m.id for m in merged] == [w.id for w in want]
        for m, w in zip(merged, want):
            np.testing.assert_array_equal(m.loc, w.loc)
            assert (m.p_c, m.f_c, m.n_points, m.n_fields) == (w.p_c, w.f_c, w.n_points, w.n_fields)
        feats_want = case.meta.get("features", {}).get(key)
        if feats_want is not None:
            got = O.features(rows, mm, case["out_point_labels"], case["out_field_labels"],
                             case["in_p_traj_id"], case["in_p_t"], case["in_p_xyz"],
                             case["in_p_value"], dims, origin, spacing, times, values)
            assert [f.id for f in got] == [f["id"] for f in feats_want]
            for g, w in zip(got, feats_want):
                assert g.member_clusters == w["member_clusters"]
                assert [list(map(int, x)) for x in g.polylines] == w["polylines"]
                assert g.isolated_points == w["isolated_points"]
                assert {str(m): list(map(int, c)) for m, c in sorted(g.voxels.items())} == w["voxels"]
                for sk, sv in w["stats"].items():
                    assert g.stats[sk] == sv, (name, g.id, sk)


def test_frontend_fixture_values():
    """The reference's recorded service responses (frontend fixtures)."""
    case = Case("run_slab2_frontend")
    fx = case.meta["frontend_fixture"]
    p = case.params
    dims, origin, spacing, times, values = case.field
    mins, maxs = case.extent
    r = O.segment(case.p_loc, case["in_p_value"], dims, origin, spacing, times, values, mins,
                  maxs, p["k"], c_f=p["c_f"], w_d=p["w_d"], w_p=p["w_p"], w_f=p["w_f"],
                  eps_c=p["eps_c"], max_iterations=p["max_iterations"])
    rows = O.table_of(r.centres)
    for row, want in zip(rows, fx["centers_all"]):
        assert row.id == want["id"]
        assert list(row.loc) == [want["x_c"], want["y_c"], want["z_c"], want["t_c"]]
        assert (row.p_c, row.f_c, row.n_points, row.n_fields) == \
            (want["p_c"], want["f_c"], want["n_points"], want["n_fields"])
    mm, merged = O.merge(rows, 2.0)
    w = fx["merge_all"]["centers"][0]
    assert {str(k): v for k, v in mm.items()} == fx["merge_all"]["merge_map"]
    assert list(merged[0].loc) == [w["x_c"], w["y_c"], w["z_c"], w["t_c"]]
    assert merged[0].p_c == w["p_c"] and merged[0].f_c == w["f_c"]
    feats = O.features(rows, None, r.point_labels, r.field_labels, case["in_p_traj_id"],
                       case["in_p_t"], case["in_p_xyz"], case["in_p_value"], dims, origin,
                       spacing, times, values)
    for k, v in fx["feature0_stats"].items():
        assert feats[0].stats[k] == v


def test_normalization_matches_reference():
    for name in ("run_slab2_frontend", "run_two_blob", "run_blob_noisy"):
        case = Case(name)
        v, lo, hi = O.minmax_normalize(case["in_raw_f_values"])
        np.testing.assert_array_equal(v, case["in_f_values"])
        assert (lo, hi) == (case.meta["normalization"]["f_min"], case.meta["normalization"]["f_max"])
        v, lo, hi = O.minmax_normalize(case["in_raw_p_value"])
        np.testing.assert_array_equal(v, case["in_p_value"])
        dims, origin, spacing, times, _ = case.field
        lo4, hi4 = O.tight_extent(case.p_loc, dims, origin, spacing, times)
        mins, maxs = case.extent
        np.testing.assert_array_equal(lo4, mins)
        np.testing.assert_array_equal(hi4, maxs)


def test_link_index_matches_reference():
    case = Case("link_blob")
    dims, origin, spacing, times, _ = case.field
    keys, sizes, members = O.link_index(dims, origin, spacing, times, case["in_p_xyz"],
                                        case["in_p_t"])
    np.testing.assert_array_equal(keys, case["out_keys"])
    np.testing.assert_array_equal(sizes, case["out_sizes"])
    np.testing.assert_array_equal(members, case["out_members"])
