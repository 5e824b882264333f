"""Run artifacts in the reference's schema (artifacts.py).

CPU: files written by the reference itself (tests/golden/artifacts_slab2, made
by `make_golden.py artifacts`) are loaded with our reader and written back
with our writer -> byte-identical.  GPU: our pipeline on the same raw inputs
writes the same files (labels byte-identical, JSON equal up to the centres'
last bits)."""
import filecmp
import json
import os

import numpy as np
import pytest

from paper_1903_12294_b200 import artifacts as A
from paper_1903_12294_b200.postproc import Feature, FeatureStats

GOLD = os.path.join(os.path.dirname(__file__), "golden", "artifacts_slab2")


def _features_from_doc(doc):
    out = []
    for f in doc["features"]:
        st = f["stats"]
        stats = FeatureStats(tuple(st["bbox_min"]), tuple(st["bbox_max"]), st["p_mean"], st["p_std"],
                             st["f_mean"], st["f_std"], st["n_points"], st["n_fields"]) if st else None
        out.append(Feature(f["id"], f["member_clusters"], [np.array(p) for p in f["polylines"]],
                           f["isolated_points"], {int(m): np.array(c) for m, c in f["voxels"].items()},
                           stats))
    return out


def test_artifacts_round_trip_byte_identical(tmp_path):
    seg, norm = A.load_segmentation(GOLD)
    A.save_segmentation(str(tmp_path), seg, norm)
    for name in (A.SEGMENTATION_JSON, A.POINT_LABELS_BIN, A.FIELD_LABELS_BIN):
        assert filecmp.cmp(os.path.join(GOLD, name), os.path.join(tmp_path, name), shallow=False), name
    eps, mm, merged = A.load_merge(GOLD)
    A.save_merge(str(tmp_path), eps, mm, merged)
    assert filecmp.cmp(os.path.join(GOLD, A.MERGE_JSON), os.path.join(tmp_path, A.MERGE_JSON),
                       shallow=False)
    doc = A.load_features(GOLD)
    A.save_features(str(tmp_path), _features_from_doc(doc), merged, mm)
    assert filecmp.cmp(os.path.join(GOLD, A.FEATURES_JSON), os.path.join(tmp_path, A.FEATURES_JSON),
                       shallow=False)


def test_artifacts_errors(tmp_path):
    with pytest.raises(A.ArtifactError):
        A.load_segmentation(str(tmp_path))
    seg, norm = A.load_segmentation(GOLD)
    A.save_segmentation(str(tmp_path), seg, norm)
    np.zeros(3, "<i4").tofile(os.path.join(tmp_path, A.POINT_LABELS_BIN))
    with pytest.raises(A.ArtifactError):
        A.load_segmentation(str(tmp_path))


def _close_json(a, b, rtol=1e-12):
    if isinstance(a, dict):
        assert a.keys() == b.keys()
        for k in a:
            _close_json(a[k], b[k], rtol)
    elif isinstance(a, list):
        assert len(a) == len(b)
        for x, y in zip(a, b):
            _close_json(x, y, rtol)
    elif isinstance(a, float) and isinstance(b, float):
        assert abs(a - b) <= rtol * max(abs(a), abs(b), 1.0), (a, b)
    else:
        assert a == b, (a, b)


@pytest.mark.gpu
def test_pipeline_artifacts_match_reference(tmp_path):
    import paper_1903_12294_b200 as P
    from golden_io import Case
    case = Case("run_slab2_frontend")
    params = P.ClusterParams.from_dict(case.meta["params"])
    raw_p = P.PointSet(case["in_p_traj_id"], case["in_p_t"], case["in_p_xyz"].reshape(-1, 3),
                       case["in_raw_p_value"])
    dims, origin, spacing, times, _ = case.field
    raw_f = P.FieldSet(dims, origin, spacing, times, case["in_raw_f_values"])
    seg, norm, _ = P.segment(raw_p, raw_f, params)
    A.save_segmentation(str(tmp_path), seg, norm)
    mm, merged = P.merge_clusters(seg.centers, 0.01)
    A.save_merge(str(tmp_path), 0.01, mm, merged)
    p_n, f_n, _ = P.normalize_variables(raw_p, raw_f, True)
    feats = P.build_features(seg, mm, p_n, f_n)
    A.save_features(str(tmp_path), feats, merged, mm)
    for name in (A.POINT_LABELS_BIN, A.FIELD_LABELS_BIN):
        assert filecmp.cmp(os.path.join(GOLD, name), os.path.join(tmp_path, name), shallow=False), name
    for name in (A.SEGMENTATION_JSON, A.MERGE_JSON, A.FEATURES_JSON):
        with open(os.path.join(GOLD, name)) as f1, open(os.path.join(tmp_path, name)) as f2:
            _close_json(json.load(f1), json.load(f2))


@pytest.mark.gpu
def test_device_run_directory_byte_identical(tmp_path, monkeypatch):
    """save_segmentation_device (labels streamed from device memory in several
    double-buffered chunks) writes the same bytes as save_segmentation of the
    host Segmentation of the same run."""
    import paper_1903_12294_b200 as P
    from paper_1903_12294_b200 import artifacts as A
    from paper_1903_12294_b200.engine import run_device
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device, synthetic_device
    from paper_1903_12294_b200.pipeline import to_segmentation
    fld, pts, _ = synthetic_device((40, 36, 30), 6, 3000, seed=8)
    norm = normalize_device(pts, fld, True)
    ext = domain_extent_device(pts, fld)
    params = P.ClusterParams(k=(4, 4, 3, 2), eps_c=1e-12, max_iterations=4)
    r = run_device(pts, fld, ext, params)
    monkeypatch.setattr(A, "_CHUNK", 10007)          # many chunks, a ragged last one
    A.save_segmentation_device(str(tmp_path / "dev"), r, params, ext, norm)
    A.save_segmentation(str(tmp_path / "host"), to_segmentation(r, params, ext), norm)
    for name in (A.SEGMENTATION_JSON, A.POINT_LABELS_BIN, A.FIELD_LABELS_BIN):
        assert (tmp_path / "dev" / name).read_bytes() == (tmp_path / "host" / name).read_bytes(), name
    seg, norm2 = A.load_segmentation(str(tmp_path / "dev"))
    assert norm2 == norm and len(seg.field_labels) == fld.values.numel()
