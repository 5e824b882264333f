"""Field files in the reference's format (ingest.py:39-106) -> device.

`load_field_device` must accept exactly what the reference's `load_field`
accepts (same validation, same errors) and produce the same f64 values:
f64 files bit for bit, f32 files widened exactly.  The metadata checks run on
CPU; the loads on the GPU.
"""
import json
import os

import numpy as np
import pytest

from paper_1903_12294_b200.ingest import IngestError, _field_meta, write_field
from paper_1903_12294_b200.model import FieldSet


def _fs(nt=3, dims=(7, 5, 4), seed=0):
    rng = np.random.default_rng(seed)
    return FieldSet(dims, np.array([0.5, -1.0, 2.0]), np.array([0.25, 1.0, 0.5]),
                    np.arange(nt, dtype=float) * 1.5, rng.random((nt, int(np.prod(dims)))))


def test_field_metadata_errors(tmp_path):
    p = tmp_path / "f.json"
    write_field(str(p), _fs())
    meta = json.loads(p.read_text())
    _field_meta(str(p))                                      # valid
    for key in ("dims", "times", "dtype", "order", "data_files"):
        bad = dict(meta)
        del bad[key]
        q = tmp_path / f"no_{key}.json"
        q.write_text(json.dumps(bad))
        with pytest.raises(IngestError, match=f"missing key '{key}'"):
            _field_meta(str(q))
    for field, value, msg in (("order", "z_fastest", "unsupported order"),
                              ("dtype", "f16", "unsupported dtype"),
                              ("times", [0.0, 2.0, 1.0], "strictly increase"),
                              ("times", [0.0, 1.0], "2 times but 3 data files")):
        bad = dict(meta)
        bad[field] = value
        q = tmp_path / "bad.json"
        q.write_text(json.dumps(bad))
        with pytest.raises(IngestError, match=msg):
            _field_meta(str(q))
    q = tmp_path / "garbage.json"
    q.write_text("{not json")
    with pytest.raises(IngestError, match="malformed"):
        _field_meta(str(q))
    with pytest.raises(FileNotFoundError):
        _field_meta(str(tmp_path / "missing.json"))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_load_field_device_matches_host_load(tmp_path, dtype):
    from paper_1903_12294_b200.ingest import load_field_device
    fs = _fs(nt=5, dims=(33, 17, 9), seed=1)
    p = tmp_path / "field.json"
    write_field(str(p), fs, dtype=dtype)
    fld = load_field_device(str(p))
    want = fs.values.astype(np.float32).astype(np.float64) if dtype == "f32" else fs.values
    np.testing.assert_array_equal(fld.values.cpu().numpy().reshape(fs.values.shape), want)
    np.testing.assert_array_equal(fld.times.cpu().numpy(), fs.times)
    assert fld.dims == fs.dims
    np.testing.assert_array_equal(fld.origin, fs.origin)


@pytest.mark.gpu
def test_load_field_device_size_and_missing_file_errors(tmp_path):
    from paper_1903_12294_b200.ingest import load_field_device
    p = tmp_path / "field.json"
    write_field(str(p), _fs(nt=3), dtype="f32")
    with open(tmp_path / "field_0001.bin", "ab") as f:
        f.write(b"\0\0\0\0")
    with pytest.raises(IngestError, match="expected 140 values"):
        load_field_device(str(p))
    os.remove(tmp_path / "field_0001.bin")
    with pytest.raises(FileNotFoundError):
        load_field_device(str(p))


@pytest.mark.gpu
def test_segment_from_files_equals_segment(tmp_path):
    """Whole pipeline from the reference's file format: the same labels and
    centres as pipeline.segment on the loaded (f32-widened) field."""
    import paper_1903_12294_b200 as P
    from paper_1903_12294_b200.ingest import synthetic_device
    fld, pts, tid = synthetic_device((24, 20, 16), 6, 300, seed=4)
    nt = 6
    fs = P.FieldSet((24, 20, 16), np.zeros(3), np.ones(3), np.arange(nt, dtype=float),
                    fld.values.cpu().numpy().reshape(nt, -1))
    ps = P.PointSet(tid.cpu().numpy(), pts.t.cpu().numpy(), pts.xyz.cpu().numpy(), pts.value.cpu().numpy())
    params = P.ClusterParams(k=(3, 3, 2, 2), eps_c=1e-12, max_iterations=4)
    write_field(str(tmp_path / "f.json"), fs, dtype="f32")
    seg, norm, _ = P.segment_from_files(str(tmp_path / "f.json"), ps, params)
    fs32 = P.FieldSet(fs.dims, fs.origin, fs.spacing, fs.times,
                      fs.values.astype(np.float32).astype(np.float64))
    ref, rnorm, _ = P.segment(ps, fs32, params)
    np.testing.assert_array_equal(seg.field_labels, ref.field_labels)
    np.testing.assert_array_equal(seg.point_labels, ref.point_labels)
    assert norm == rnorm


@pytest.mark.gpu
def test_segment_to_dir_from_files(tmp_path):
    """Files in -> run directory out (labels streamed from the device): the
    deterministic files equal save_segmentation of pipeline.segment's result;
    report.json has the reference's keys plus the throughput keys."""
    import paper_1903_12294_b200 as P
    from paper_1903_12294_b200 import artifacts as A
    from paper_1903_12294_b200.ingest import synthetic_device
    from paper_1903_12294_b200.pipeline import segment_to_dir
    fld, pts, tid = synthetic_device((20, 18, 14), 5, 250, seed=9)
    nt = 5
    fs = P.FieldSet((20, 18, 14), np.zeros(3), np.ones(3), np.arange(nt, dtype=float),
                    fld.values.cpu().numpy().reshape(nt, -1))
    ps = P.PointSet(tid.cpu().numpy(), pts.t.cpu().numpy(), pts.xyz.cpu().numpy(), pts.value.cpu().numpy())
    params = P.ClusterParams(k=(3, 3, 2, 2), eps_c=1e-12, max_iterations=4)
    write_field(str(tmp_path / "in" / "f.json"), fs, dtype="f64")
    segment_to_dir(str(tmp_path / "dev"), str(tmp_path / "in" / "f.json"), ps, params)
    seg, norm, _ = P.segment(ps, fs, params)
    A.save_segmentation(str(tmp_path / "host"), seg, norm)
    for name in (A.SEGMENTATION_JSON, A.POINT_LABELS_BIN, A.FIELD_LABELS_BIN):
        assert (tmp_path / "dev" / name).read_bytes() == (tmp_path / "host" / name).read_bytes(), name
    rep = A.load_report(str(tmp_path / "dev"))
    for key in ("inputs", "params", "n_point_samples", "n_field_samples", "iterations_used",
                "converged", "iteration_seconds", "total_seconds", "voxel_timesteps_per_s", "passes"):
        assert key in rep, key
    assert len(rep["iteration_seconds"]) == rep["iterations_used"]


@pytest.mark.gpu
@pytest.mark.parametrize("n,dtype", [(123_456_789, "int32"), (9_999_991, "float64"), (1000, "int32")])
def test_staged_transfers_round_trip(n, dtype):
    """Pageable arrays through the pinned staging ring (engine._Stager): upload
    (to_dev) and download (engine.download, with on-device int32 -> int64
    widening) reproduce the bytes, also for sizes that are not a multiple of the
    32 MB slot and below the staging threshold."""
    import torch
    from paper_1903_12294_b200.engine import download, to_dev
    rng = np.random.default_rng(n)
    a = (rng.integers(-2**31, 2**31 - 1, n, dtype=np.int64).astype(np.int32) if dtype == "int32"
         else rng.standard_normal(n))
    d = to_dev(a, torch.int32 if dtype == "int32" else torch.float64)
    assert np.array_equal(d.cpu().numpy(), a)
    np.testing.assert_array_equal(download(d), a)
    if dtype == "int32":
        w = download(d, torch.int64)
        assert w.dtype == np.int64
        np.testing.assert_array_equal(w, a.astype(np.int64))
