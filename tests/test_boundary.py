"""Hardening of the drop-in boundary.

* Non-finite inputs are rejected with ValueError instead of
  silently diverging from numpy (whose min/argmin propagate NaN).
* Inputs whose per-cluster sums could overflow the exact 128-bit fixed-point
  accumulators are rejected instead of wrapping.
* The degenerate-range normalisation maps to zeros with a UserWarning
  (ingest.py:312-318).
* `segment()` works from a non-main thread (the reference's service runs it on
  a daemon thread, service.py:137-155).
* Objects that are not this package's value types but carry the reference's
  attributes (model.py:78-157) are accepted: `RefPointSet` / `RefFieldSet`
  below restate the reference dataclasses' fields, and a CPU test checks that
  restatement against the reference's own classes when /root/reference exists.
* The C ABI accepts a workspace pointer of any alignment.
"""
import dataclasses
import os
import sys
import threading
import warnings

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"


@dataclasses.dataclass(frozen=True)
class RefPointSet:
    """Attribute clone of the reference's mfseg.model.PointSet (model.py:78-105)."""
    traj_id: np.ndarray
    t: np.ndarray
    xyz: np.ndarray
    value: np.ndarray

    def __len__(self):
        return len(self.traj_id)


@dataclasses.dataclass(frozen=True)
class RefFieldSet:
    """Attribute clone of the reference's mfseg.model.FieldSet (model.py:108-157)."""
    dims: tuple
    origin: np.ndarray
    spacing: np.ndarray
    times: np.ndarray
    values: np.ndarray

    def __len__(self):
        return int(np.prod(self.dims)) * len(self.times)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")
def test_clones_match_reference_value_types():
    sys.path.insert(0, REF_SRC)
    try:
        from mfseg import model as R
    finally:
        sys.path.remove(REF_SRC)
    for ref, clone in ((R.PointSet, RefPointSet), (R.FieldSet, RefFieldSet)):
        assert [f.name for f in dataclasses.fields(ref)] == [f.name for f in dataclasses.fields(clone)]
    from paper_1903_12294_b200 import model as M
    for name in ("PointSet", "FieldSet", "DomainExtent", "ClusterParams", "ClusterCenter",
                 "Segmentation"):
        assert ([f.name for f in dataclasses.fields(getattr(R, name))] ==
                [f.name for f in dataclasses.fields(getattr(M, name))]), name


def _small(seed=0, nt=4, dims=(12, 10, 8), ntraj=60):
    from paper_1903_12294_b200.ingest import synthetic_device
    fld, pts, tid = synthetic_device(dims, nt, ntraj, seed=seed, noise=0.05, n_blobs=3)
    fv = fld.values.cpu().numpy().reshape(nt, -1)
    ps = RefPointSet(tid.cpu().numpy(), pts.t.cpu().numpy(), pts.xyz.cpu().numpy(),
                     pts.value.cpu().numpy())
    fs = RefFieldSet(dims, np.zeros(3), np.ones(3), np.arange(nt, dtype=float), fv)
    return ps, fs


@pytest.mark.gpu
def test_reference_like_objects_are_accepted():
    import paper_1903_12294_b200 as P
    ps, fs = _small(1)
    params = P.ClusterParams(k=(3, 2, 2, 2), eps_c=1e-12, max_iterations=4)
    seg, norm, _ = P.segment(ps, fs, params)
    ours = P.PointSet(ps.traj_id, ps.t, ps.xyz, ps.value)
    ourf = P.FieldSet(fs.dims, fs.origin, fs.spacing, fs.times, fs.values)
    ref, norm2, _ = P.segment(ours, ourf, params)
    np.testing.assert_array_equal(seg.field_labels, ref.field_labels)
    np.testing.assert_array_equal(seg.point_labels, ref.point_labels)
    assert norm == norm2


@pytest.mark.gpu
@pytest.mark.parametrize("where", ["field_value", "point_value", "point_xyz", "point_t", "field_time"])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("normalize", [True, False])
def test_non_finite_inputs_rejected(where, bad, normalize):
    import paper_1903_12294_b200 as P
    ps, fs = _small(2)
    fv, pv, xyz, t, times = (fs.values.copy(), ps.value.copy(), ps.xyz.copy(), ps.t.copy(),
                             fs.times.copy())
    {"field_value": lambda: fv.__setitem__((1, 37), bad),
     "point_value": lambda: pv.__setitem__(5, bad),
     "point_xyz": lambda: xyz.__setitem__((7, 1), bad),
     "point_t": lambda: t.__setitem__(9, bad),
     "field_time": lambda: times.__setitem__(-1, bad if bad != -np.inf else np.inf)}[where]()
    ps2 = RefPointSet(ps.traj_id, t, xyz, pv)
    fs2 = RefFieldSet(fs.dims, fs.origin, fs.spacing, times, fv)
    params = P.ClusterParams(k=(3, 2, 2, 2), max_iterations=2, normalize=normalize)
    with pytest.raises(ValueError):
        P.segment(ps2, fs2, params)


@pytest.mark.gpu
def test_sum_range_overflow_rejected():
    """|x| * n >= 2^62 could wrap the 128-bit accumulators: rejected up front."""
    import paper_1903_12294_b200 as P
    ps, fs = _small(3)
    xyz = ps.xyz.copy()
    xyz[:, 0] += 1e17            # 480 point samples * 1e17 > 2^62 = 4.6e18
    ps2 = RefPointSet(ps.traj_id, ps.t, xyz, ps.value)
    params = P.ClusterParams(k=(3, 2, 2, 2), max_iterations=2)
    with pytest.raises(ValueError, match="too large"):
        P.segment(ps2, None, params)
    ok = xyz.copy()
    ok[:, 0] -= 1e17 - 1e14      # 480 * 1e14 fits
    P.segment(RefPointSet(ps.traj_id, ps.t, ok, ps.value), None, params)


@pytest.mark.gpu
def test_degenerate_range_normalises_to_zero_with_warning():
    """ingest.py:312-318: hi == lo -> zeros and a UserWarning, per kind."""
    import paper_1903_12294_b200 as P
    ps, fs = _small(4)
    fs2 = RefFieldSet(fs.dims, fs.origin, fs.spacing, fs.times, np.full_like(fs.values, 0.25))
    params = P.ClusterParams(k=(3, 2, 2, 2), eps_c=1e-12, max_iterations=3)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        seg, norm, _ = P.segment(ps, fs2, params)
    assert any("degenerate" in str(x.message) for x in w)
    assert norm.f_min == norm.f_max == 0.25
    # the field contributes value 0 everywhere: every field centre value is 0
    assert all(c.f_c == 0.0 for c in seg.centers if c.f_c is not None)
    # and the labels equal a run on an all-zero field without normalisation
    fs0 = RefFieldSet(fs.dims, fs.origin, fs.spacing, fs.times, np.zeros_like(fs.values))
    pv = (ps.value - ps.value.min()) / (ps.value.max() - ps.value.min())   # ingest.py:312-318
    seg0, _, _ = P.segment(RefPointSet(ps.traj_id, ps.t, ps.xyz, pv), fs0,
                           P.ClusterParams(k=(3, 2, 2, 2), eps_c=1e-12, max_iterations=3,
                                           normalize=False))
    np.testing.assert_array_equal(seg.field_labels, seg0.field_labels)


@pytest.mark.gpu
def test_segment_from_non_main_thread():
    import paper_1903_12294_b200 as P
    ps, fs = _small(5)
    params = P.ClusterParams(k=(3, 2, 2, 2), eps_c=1e-12, max_iterations=4)
    ref, _, _ = P.segment(ps, fs, params)
    out = {}

    def job():
        try:
            out["seg"] = P.segment(ps, fs, params)[0]
        except BaseException as e:   # surfaced below
            out["err"] = e

    th = threading.Thread(target=job, daemon=True)
    th.start()
    th.join(120)
    assert "err" not in out, out.get("err")
    np.testing.assert_array_equal(out["seg"].field_labels, ref.field_labels)
    np.testing.assert_array_equal(out["seg"].point_labels, ref.point_labels)


@pytest.mark.gpu
def test_misaligned_workspace():
    """The workspace pointer may have any alignment (the carvings align themselves)."""
    import torch
    import paper_1903_12294_b200 as P
    from paper_1903_12294_b200.engine import run_device
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device, synthetic_device
    fld, pts, _ = synthetic_device((16, 12, 10), 4, 80, seed=6)
    normalize_device(pts, fld, True)
    ext = domain_extent_device(pts, fld)
    params = P.ClusterParams(k=(3, 2, 2, 2), eps_c=1e-12, max_iterations=3)
    a = run_device(pts, fld, ext, params)
    big = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    b = run_device(pts, fld, ext, params, workspace=big[13:])
    assert torch.equal(a.field_labels, b.field_labels)
    assert torch.equal(a.point_labels, b.point_labels)
