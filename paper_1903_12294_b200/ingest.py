"""GPU-backed parts of the reference's `mfseg.ingest` that sit on the hot path.

  normalize_variables  min-max per kind on the device (ingest.py:312-335)
  domain_extent        tight 4D box; point min/max reduced on the device
                       (ingest.py:204-227)
  build_link_index     (cell, interval) buckets via a stable device radix sort
                       (ingest.py:261-280)
  synthetic_*          counter-based benchmark inputs generated on the device

File formats, CSV parsing and derivation expressions are out of scope (host
I/O); callers hand in arrays.
"""

from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .engine import DeviceField, DevicePoints, device, stream_ptr, to_dev
from .model import DomainExtent, FieldSet, PointSet


class IngestError(ValueError):
    """Malformed or inconsistent input data (ingest.py:28-29)."""


@dataclass(frozen=True)
class NormalizationRecord:
    """Min/max per kind (ingest.py:293-309)."""

    enabled: bool
    p_min: Optional[float] = None
    p_max: Optional[float] = None
    f_min: Optional[float] = None
    f_max: Optional[float] = None

    def to_dict(self) -> dict:
        return {"enabled": self.enabled, "p_min": self.p_min, "p_max": self.p_max,
                "f_min": self.f_min, "f_max": self.f_max}

    @classmethod
    def from_dict(cls, d: dict) -> "NormalizationRecord":
        return cls(**d)


def minmax_normalize_(values: torch.Tensor, kind: str, apply: bool = True):
    """In place (v - lo)/(hi - lo) on a device tensor; degenerate -> zeros + warning."""
    lib = N.load()
    lo, hi = C.c_double(0.0), C.c_double(0.0)
    N.check(lib.mfseg_minmax_normalize(N.ptr(values), values.numel(), int(apply), C.byref(lo),
                                       C.byref(hi), stream_ptr()), "mfseg_minmax_normalize")
    if apply and hi.value == lo.value:
        warnings.warn(f"{kind} variable has a degenerate range ({lo.value}); all values map to 0")
    return float(lo.value), float(hi.value)


def normalize_device(pts: DevicePoints, fld: DeviceField, enabled: bool) -> NormalizationRecord:
    """normalize_variables on device-resident data (in place)."""
    if not enabled:
        return NormalizationRecord(enabled=False)
    p_min = p_max = f_min = f_max = None
    if pts.n > 0:
        p_min, p_max = minmax_normalize_(pts.value, "point")
    if fld.values.numel() > 0:
        f_min, f_max = minmax_normalize_(fld.values, "field")
    return NormalizationRecord(True, p_min, p_max, f_min, f_max)


def normalize_variables(points: Optional[PointSet], fs: Optional[FieldSet], enabled: bool):
    """Min-max map v_p and v_f independently onto [0, 1] (ingest.py:321-335)."""
    if not enabled:
        return points, fs, NormalizationRecord(enabled=False)
    dev = device()
    p_min = p_max = f_min = f_max = None
    if points is not None and len(points) > 0:
        v = to_dev(points.value, dev=dev)
        p_min, p_max = minmax_normalize_(v, "point")
        points = PointSet(points.traj_id, points.t, points.xyz, v.cpu().numpy())
    if fs is not None and len(fs) > 0:
        v = to_dev(np.asarray(fs.values).reshape(-1), dev=dev)
        f_min, f_max = minmax_normalize_(v, "field")
        fs = FieldSet(fs.dims, fs.origin, fs.spacing, fs.times,
                      v.cpu().numpy().reshape(np.asarray(fs.values).shape))
    return points, fs, NormalizationRecord(True, p_min, p_max, f_min, f_max)


def _extent_from(lo_parts, hi_parts, pad):
    if not lo_parts:
        raise IngestError("no samples: cannot derive a domain extent")
    lo = np.min(lo_parts, axis=0)
    hi = np.max(hi_parts, axis=0)
    span = hi - lo
    hi = np.where(span <= 0, hi + np.maximum(pad, np.abs(hi) * pad) + pad, hi)
    return DomainExtent(lo[0], hi[0], lo[1], hi[1], lo[2], hi[2], lo[3], hi[3])


def domain_extent_device(pts: DevicePoints, fld: DeviceField, pad: float = 1e-9) -> DomainExtent:
    """Tight 4D bounding region (ingest.py:204-227)."""
    los, his = [], []
    if fld.nt > 0:
        t = fld.times
        t0, t1 = (float(x) for x in torch.stack([t[0], t[-1]]).cpu())
        los.append(np.concatenate([fld.origin, [t0]]))
        his.append(np.concatenate([fld.origin + np.array(fld.dims) * fld.spacing, [t1]]))
    if pts.n > 0:
        mn = torch.cat([pts.xyz.amin(dim=0), pts.t.amin().reshape(1)])
        mx = torch.cat([pts.xyz.amax(dim=0), pts.t.amax().reshape(1)])
        los.append(mn.cpu().numpy())
        his.append(mx.cpu().numpy())
    return _extent_from(los, his, pad)


def domain_extent(points: Optional[PointSet], fs: Optional[FieldSet], pad: float = 1e-9):
    from .engine import field_to_device, points_to_device
    dev = device()
    return domain_extent_device(points_to_device(points, dev), field_to_device(fs, dev), pad)


@dataclass(frozen=True)
class LinkIndex:
    """Point indices bucketed by (i, j, k, m) (ingest.py:246-258)."""

    buckets: dict

    def total_points(self) -> int:
        return sum(len(v) for v in self.buckets.values())


def link_index_device(fld: DeviceField, pts: DevicePoints):
    """Device CSR form: (sorted flat keys int64, members int32, n_buckets)."""
    lib = N.load()
    dev = pts.t.device
    n = pts.n
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    members = torch.empty(n, dtype=torch.int32, device=dev)
    nb = C.c_int64(0)
    ws_bytes = lib.mfseg_link_index_workspace_size(n)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    fs, ps = fld.struct(), pts.struct()
    rc = lib.mfseg_link_index(C.byref(fs), C.byref(ps), N.ptr(keys), N.ptr(members),
                              C.byref(nb), N.ptr(ws), ws_bytes, stream_ptr())
    if rc == 2:
        raise IngestError(lib.mfseg_last_error().decode())
    N.check(rc, "mfseg_link_index")
    return keys, members, int(nb.value)


def build_link_index(fs: FieldSet, points: PointSet) -> LinkIndex:
    """Bucket every point sample into its containing cell and time interval."""
    if len(points) == 0:
        return LinkIndex({})
    from .engine import field_to_device, points_to_device
    dev = device()
    fld, pts = field_to_device(fs, dev), points_to_device(points, dev)
    keys, members, _ = link_index_device(fld, pts)
    keys = keys.cpu().numpy()
    members = members.cpu().numpy().astype(np.int64)
    nx, ny, _ = fs.dims
    n_int = max(len(fs.times) - 1, 1)
    cut = np.flatnonzero(np.r_[True, keys[1:] != keys[:-1]])
    ends = np.r_[cut[1:], len(keys)]
    out = {}
    for a, e in zip(cut, ends):
        key = int(keys[a])
        k3, m = divmod(key, n_int)
        out[(k3 % nx, (k3 // nx) % ny, k3 // (nx * ny), m)] = members[a:e]
    return LinkIndex(out)


# ============================================================== synthetic inputs

def synth_spec(dims, nt, n_traj, seed=0, noise=0.05, n_blobs=6, dyadic=False) -> N.Synth:
    s = N.Synth()
    s.nx, s.ny, s.nz = (int(d) for d in dims)
    s.nt = int(nt)
    s.n_traj = int(n_traj)
    s.seed = int(seed)
    s.noise = float(noise)
    s.n_blobs = int(n_blobs)
    s.dyadic = int(bool(dyadic))
    return s


def synthetic_device(dims, nt, n_traj, seed=0, noise=0.05, n_blobs=6, dyadic=False, dev=None):
    """(DeviceField, DevicePoints, traj_id) of the counter-based generator.
    Grid origin 0, spacing 1, times 0..nt-1; one point sample per trajectory
    and timestep, trajectory-major (like the reference's generator)."""
    lib = N.load()
    dev = dev or device()
    s = synth_spec(dims, nt, n_traj, seed, noise, n_blobs, dyadic)
    ncell = int(np.prod(dims))
    values = torch.empty(ncell * nt, dtype=torch.float64, device=dev)
    N.check(lib.mfseg_synth_field(C.byref(s), N.ptr(values), stream_ptr()), "mfseg_synth_field")
    n = int(n_traj) * int(nt)
    tid = torch.empty(n, dtype=torch.int64, device=dev)
    t = torch.empty(n, dtype=torch.float64, device=dev)
    xyz = torch.empty((n, 3), dtype=torch.float64, device=dev)
    v = torch.empty(n, dtype=torch.float64, device=dev)
    if n:
        N.check(lib.mfseg_synth_points(C.byref(s), N.ptr(tid), N.ptr(t), N.ptr(xyz), N.ptr(v),
                                       stream_ptr()), "mfseg_synth_points")
    fld = DeviceField(tuple(int(d) for d in dims), np.zeros(3), np.ones(3),
                      torch.arange(nt, dtype=torch.float64, device=dev), values)
    return fld, DevicePoints(xyz, t, v), tid


def synthetic_field_window(dims, nt, seed=0, noise=0.05, n_blobs=6, dyadic=False, dev=None,
                           m0=0, m1=None, z0=0, z1=None) -> DeviceField:
    """Timesteps [m0, m1) x z-planes [z0, z1) of `synthetic_device`'s field (a
    time or spatial slab; values bit-identical to the whole dataset's)."""
    lib = N.load()
    dev = dev or device()
    m1 = nt if m1 is None else m1
    z1 = dims[2] if z1 is None else z1
    s = synth_spec(dims, nt, 0, seed, noise, n_blobs, dyadic)
    values = torch.empty(int(dims[0]) * int(dims[1]) * (z1 - z0) * (m1 - m0), dtype=torch.float64,
                         device=dev)
    N.check(lib.mfseg_synth_field_window(C.byref(s), m0, m1, z0, z1, N.ptr(values), stream_ptr()),
            "mfseg_synth_field_window")
    return DeviceField((int(dims[0]), int(dims[1]), z1 - z0), np.zeros(3), np.ones(3),
                       torch.arange(m0, m1, dtype=torch.float64, device=dev), values, (0, 0, z0))


def synthetic_points_window(dims, nt, n_traj, seed=0, noise=0.05, n_blobs=6, dyadic=False,
                            dev=None, m0=0, m1=None, keep=None, chunk=1 << 22):
    """Point samples of `synthetic_device` at timesteps [m0, m1) (all
    trajectories, trajectory-major), optionally only those for which
    keep(xyz, t) (a device mask function, e.g. a z-bin range) holds; generated in
    chunks of trajectories so a slab never materialises the whole set.
    Returns (DevicePoints, traj_id)."""
    lib = N.load()
    dev = dev or device()
    m1 = nt if m1 is None else m1
    s = synth_spec(dims, nt, n_traj, seed, noise, n_blobs, dyadic)
    w = m1 - m0
    parts = []
    for p0 in range(0, int(n_traj), chunk if keep is not None else max(int(n_traj), 1)):
        p1 = min(int(n_traj), p0 + (chunk if keep is not None else int(n_traj)))
        n = (p1 - p0) * w
        tid = torch.empty(n, dtype=torch.int64, device=dev)
        t = torch.empty(n, dtype=torch.float64, device=dev)
        xyz = torch.empty((n, 3), dtype=torch.float64, device=dev)
        v = torch.empty(n, dtype=torch.float64, device=dev)
        if n:
            N.check(lib.mfseg_synth_points_window(C.byref(s), p0, p1, m0, m1, N.ptr(tid), N.ptr(t),
                                                  N.ptr(xyz), N.ptr(v), stream_ptr()),
                    "mfseg_synth_points_window")
        if keep is not None:
            sel = keep(xyz, t)
            tid, t, xyz, v = tid[sel], t[sel], xyz[sel], v[sel]
        parts.append((tid, t, xyz, v))
    if not parts:
        z = torch.zeros(0, dtype=torch.float64, device=dev)
        return DevicePoints(z.reshape(0, 3), z, z), torch.zeros(0, dtype=torch.int64, device=dev)
    if len(parts) == 1:
        tid, t, xyz, v = parts[0]
    else:
        tid, t, xyz, v = (torch.cat([p[i] for p in parts]) for i in range(4))
    return DevicePoints(xyz.contiguous(), t.contiguous(), v.contiguous()), tid


def synthetic_taxi_points(dims, nt, n_traj, steps=8, skew=0.7, road_frac=0.02, seed=0, noise=0.05,
                          n_blobs=6, dev=None, p0=0, p1=None):
    """configs[3]'s taxi-like trajectories (2D+t, nz = 1): `steps` consecutive
    samples per trajectory from a uniform random start, a fraction `skew` of
    them on `road_frac` of the rows / columns.  Returns (DevicePoints, traj_id)."""
    lib = N.load()
    dev = dev or device()
    p1 = n_traj if p1 is None else p1
    s = synth_spec(dims, nt, n_traj, seed, noise, n_blobs, False)
    n = (p1 - p0) * steps
    tid = torch.empty(n, dtype=torch.int64, device=dev)
    t = torch.empty(n, dtype=torch.float64, device=dev)
    xyz = torch.empty((n, 3), dtype=torch.float64, device=dev)
    v = torch.empty(n, dtype=torch.float64, device=dev)
    N.check(lib.mfseg_synth_taxi_points(C.byref(s), steps, skew, road_frac, p0, p1, N.ptr(tid),
                                        N.ptr(t), N.ptr(xyz), N.ptr(v), stream_ptr()),
            "mfseg_synth_taxi_points")
    return DevicePoints(xyz, t, v), tid


# ============================================================== field files -> device

FIELD_DTYPES = {"f32": "<f4", "f64": "<f8"}   # ingest.py:25


def _field_meta(path: str):
    """Metadata document of a field (ingest.py:39-64), validated like the
    reference: same keys, order, dtype and time checks, same errors."""
    import json
    import os
    try:
        with open(path) as f:
            meta = json.load(f)
    except FileNotFoundError:
        raise
    except (json.JSONDecodeError, UnicodeDecodeError) as e:
        raise IngestError(f"{path}: malformed field metadata: {e}")
    for key in ("dims", "origin", "spacing", "times", "variable", "data_files", "dtype", "order"):
        if key not in meta:
            raise IngestError(f"{path}: metadata missing key '{key}'")
    if meta["order"] != "x_fastest":
        raise IngestError(f"{path}: unsupported order '{meta['order']}'")
    if meta["dtype"] not in FIELD_DTYPES:
        raise IngestError(f"{path}: unsupported dtype '{meta['dtype']}'")
    dims = tuple(int(d) for d in meta["dims"])
    times = np.asarray(meta["times"], dtype=float)
    if len(times) != len(meta["data_files"]):
        raise IngestError(f"{path}: {len(times)} times but {len(meta['data_files'])} data files")
    if len(times) > 1 and not np.all(np.diff(times) > 0):
        raise IngestError(f"{path}: timestep times must strictly increase")
    base = os.path.dirname(os.path.abspath(path))
    files = [os.path.join(base, fname) for fname in meta["data_files"]]
    return meta, dims, times, files, np.dtype(FIELD_DTYPES[meta["dtype"]])


def load_field_device(path: str, dev=None) -> DeviceField:
    """load_field (ingest.py:39-78) straight into device memory.

    Each timestep's raw file is read into one of two pinned buffers while the
    copy engine moves the other one to the device (file reads overlap the
    PCIe transfer; no pageable host copy of the whole field exists).  f32 files
    cross PCIe as f32 and are widened on the device (exact, like the
    reference's `astype(np.float64)`).  Errors match the reference's."""
    import os
    meta, dims, times, files, dtype = _field_meta(path)
    dev = dev or device()
    ncell = dims[0] * dims[1] * dims[2]
    nt = len(times)
    values = torch.empty(nt * ncell, dtype=torch.float64, device=dev)
    tdtype = torch.float32 if dtype.itemsize == 4 else torch.float64
    nbytes = ncell * dtype.itemsize
    bufs = [torch.empty(ncell, dtype=tdtype, pin_memory=True) for _ in range(min(2, nt))]
    done = [torch.cuda.Event() for _ in bufs]
    stage = torch.empty(ncell, dtype=tdtype, device=dev) if tdtype != torch.float64 else None
    stream = torch.cuda.current_stream(dev)
    for m, fpath in enumerate(files):
        b = m % len(bufs)
        if m >= len(bufs):
            done[b].synchronize()           # the DMA out of this buffer has finished
        with open(fpath, "rb") as f:            # missing file: FileNotFoundError, as np.fromfile
            size = os.fstat(f.fileno()).st_size
            if size != nbytes:
                got = size // dtype.itemsize
                raise IngestError(f"{fpath}: expected {ncell} values ({nbytes} bytes), "
                                  f"got {got} (byte offset {got * dtype.itemsize})")
            f.readinto(memoryview(bufs[b].numpy()).cast("B"))
        dst = values[m * ncell:(m + 1) * ncell]
        if stage is None:
            dst.copy_(bufs[b], non_blocking=True)
        else:
            stage.copy_(bufs[b], non_blocking=True)
            dst.copy_(stage)                # f32 -> f64 widening on the device
        done[b].record(stream)
    for e in done:
        e.synchronize()
    return DeviceField(dims, np.asarray(meta["origin"], dtype=float),
                       np.asarray(meta["spacing"], dtype=float),
                       torch.as_tensor(times, dtype=torch.float64, device=dev), values)


def write_field(path: str, fs: FieldSet, variable: str = "v", dtype: str = "f64") -> None:
    """The reference's field format (ingest.py:83-106): metadata sidecar + one
    raw little-endian array per timestep."""
    import json
    import os
    if dtype not in FIELD_DTYPES:
        raise IngestError(f"unsupported dtype '{dtype}'")
    base = os.path.dirname(os.path.abspath(path))
    os.makedirs(base, exist_ok=True)
    stem = os.path.splitext(os.path.basename(path))[0]
    data_files = [f"{stem}_{m:04d}.bin" for m in range(len(fs.times))]
    meta = {"dims": list(fs.dims), "origin": [float(v) for v in fs.origin],
            "spacing": [float(v) for v in fs.spacing], "times": [float(t) for t in fs.times],
            "variable": variable, "data_files": data_files, "dtype": dtype, "order": "x_fastest"}
    np_dtype = np.dtype(FIELD_DTYPES[dtype])
    values = np.asarray(fs.values)
    for m, fname in enumerate(data_files):
        values[m].astype(np_dtype).tofile(os.path.join(base, fname))
    with open(path, "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
        f.write("\n")
