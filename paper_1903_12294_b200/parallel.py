"""Multi-GPU segmentation: whole-bin slabs across ranks, one exact exchange per pass.

The reference is single-process; the paper sketches
per-iteration centre merging across GPUs as future work.
Given the (replicated) centres every sample's label is independent, so the
samples are partitioned and the only data-path collective is, once per pass, a
SUM all-reduce of the per-cluster partial sums.  Two partitions:

* time slabs (configs[2]): every rank owns a contiguous run of field
  timesteps whose boundaries fall on t-bin changes, plus the point samples whose
  t-bin lies in its bin range;
* spatial z-slabs (configs[4]): every rank owns a contiguous run of z-planes
  whose boundaries fall on z-bin changes (the field keeps the grid's origin and
  records the slab's first global plane in `DeviceField.offset`, so every cell
  centre rounds exactly as the reference's `origin + (k + 0.5) * spacing`), plus
  the point samples whose z-bin lies in its bin range.

Whole bins per rank keep every field block and point chunk (the kernels' units
of fixed-order summation, both confined to one 4D sample bin) on one GPU, and the
partial sums are 128-bit fixed-point integers exchanged as three 42-bit limbs
per word, so the reduced sums -- and therefore centres and labels -- are
bit-identical for any number of ranks.

Host-side pieces (slab split, bin ranges, point selection, min/max and extent
agreement, the limb all-reduce, the sharded feature statistics and trajectory
stitching of `build_features_sharded`) are plain torch.distributed and numpy,
exercised on CPU with gloo by tests/test_parallel.py.
"""

from __future__ import annotations

import ctypes as C
import time
import warnings
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .engine import DeviceField, DevicePoints, run_device, stream_ptr
from .model import DomainExtent

# ============================================================== slab geometry


def time_slab(rank: int, world: int, nt: int):
    """[m0, m1) timestep range of `rank` (contiguous, sizes differ by <= 1)."""
    base, extra = divmod(nt, world)
    m0 = rank * base + min(rank, extra)
    return m0, m0 + base + (1 if rank < extra else 0)


def bins_of(x, lo: float, C: float, k: int):
    """clip(floor((x - lo) / C), 0, k - 1) (engine.py:111-113), numpy or torch."""
    if isinstance(x, torch.Tensor):
        return torch.clamp(torch.floor((x - lo) / C), 0, k - 1).to(torch.int64)
    x = np.asarray(x, dtype=np.float64)
    return np.clip(np.floor((x - lo) / C), 0, k - 1).astype(np.int64)


def bin_slabs(coords, lo: float, C: float, k: int, world: int):
    """Contiguous index slabs [i0, i1) per rank over a sorted 1-D coordinate list
    (field timesteps or cell centres along one axis) whose boundaries fall on bin
    changes, as balanced as the bin boundaries allow."""
    b = bins_of(coords, lo, C, k)
    n = len(b)
    cuts = np.flatnonzero(b[1:] != b[:-1]) + 1          # allowed slab starts
    bounds = [0]
    for r in range(1, world):
        target = r * n / world
        ok = cuts[cuts >= bounds[-1]]
        bounds.append(int(ok[np.argmin(np.abs(ok - target))]) if len(ok) else n)
    bounds.append(n)
    return [(bounds[r], max(bounds[r], bounds[r + 1])) for r in range(world)]


def tbin_slabs(times, t_min: float, C_t: float, k_t: int, world: int):
    """Timestep slabs [m0, m1) of whole t-bins (engine.py:111-113)."""
    return bin_slabs(np.asarray(times, dtype=np.float64), t_min, C_t, k_t, world)


def cell_centres(n: int, origin: float, spacing: float) -> np.ndarray:
    """origin + (i + 0.5) * spacing with the reference's two roundings (model.py:137-142)."""
    return origin + (np.arange(n, dtype=np.float64) + 0.5) * spacing


def zbin_slabs(nz: int, origin_z: float, spacing_z: float, z_min: float, C_z: float, k_z: int,
               world: int):
    """z-plane slabs [k0, k1) of whole z-bins."""
    return bin_slabs(cell_centres(nz, origin_z, spacing_z), z_min, C_z, k_z, world)


def slab_bin_ranges(coords, lo: float, C: float, k: int, slabs):
    """Bin range [b0, b1) owned by each rank: from the bin of its slab's first
    coordinate to the next non-empty slab's (rank 0 from bin 0, the last
    non-empty rank up to k), so that every bin -- also bins no field sample
    occupies -- has exactly one owner for the point samples."""
    b = bins_of(coords, lo, C, k)
    firsts = [int(b[i0]) if i1 > i0 else None for i0, i1 in slabs]
    out = []
    nonempty = [r for r, f in enumerate(firsts) if f is not None]
    for r, f in enumerate(firsts):
        if f is None:
            out.append((0, 0))
            continue
        b0 = 0 if r == nonempty[0] else f
        later = [firsts[q] for q in nonempty if q > r]
        out.append((b0, later[0] if later else k))
    return out


def select_points_for_slab(coord, lo: float, C: float, k: int, b0: int, b1: int):
    """Mask of the point samples whose bin along the sharded axis lies in [b0, b1)."""
    b = bins_of(coord, lo, C, k)
    return (b >= b0) & (b < b1)


# ============================================================== collectives


def global_minmax(lo: float, hi: float, group=None, device=None):
    """Exact global (min, max) of per-rank values (inf/-inf for empty ranks)."""
    t = torch.tensor([lo, -hi], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return float(t[0]), float(-t[1])


def global_sum_int(x: int, group=None, device=None) -> int:
    t = torch.tensor([int(x)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def allreduce_limbs(limbs: torch.Tensor, group=None) -> None:
    """In-place SUM of int64 limb words across ranks (exact: each limb < 2^42)."""
    dist.all_reduce(limbs, op=dist.ReduceOp.SUM, group=group)


def _value_range(vals: torch.Tensor):
    """(min, max, non-finite?) of a device column; (inf, -inf, False) when empty."""
    if not vals.numel():
        return float("inf"), float("-inf"), False
    lo, hi = float(vals.amin()), float(vals.amax())
    return lo, hi, bool(np.isnan(lo) or np.isnan(hi) or lo == -np.inf or hi == np.inf)


def normalize_and_extent_sharded(pts: DevicePoints, fld: DeviceField, enabled: bool = True,
                                 group=None, grid_dims=None, pad: float = 1e-9):
    """normalize_variables + domain_extent over the union of all ranks' slabs
    (ingest.py:204-227, 312-335): identical to the single-GPU result.

    `grid_dims`: the whole grid's dims when `fld` is a spatial slab (default:
    fld.dims).  Returns (DomainExtent, NormalizationRecord).  Non-finite values
    raise ValueError, as does a data range the exact 128-bit
    cluster sums cannot hold (max |x| * samples >= 2^62 over all ranks)."""
    from .ingest import NormalizationRecord
    lib = N.load()
    dev = fld.values.device if fld.values.numel() else pts.t.device
    rng = {}
    vmax = {}
    for kind, vals in (("point", pts.value), ("field", fld.values)):
        lo, hi, bad = _value_range(vals)
        if global_sum_int(bad, group, dev):
            raise ValueError(f"non-finite (NaN or inf) {kind} value")
        glo, ghi = global_minmax(lo, hi, group, dev)
        rng[kind] = (glo, ghi)
        if enabled and vals.numel() and np.isfinite(glo):
            if ghi == glo:
                warnings.warn(f"{kind} variable has a degenerate range ({glo}); all values map to 0")
            N.check(lib.mfseg_normalize_range(N.ptr(vals), vals.numel(), glo, ghi, stream_ptr()),
                    "mfseg_normalize_range")
        vmax[kind] = (1.0 if enabled else max(abs(glo), abs(ghi))) if np.isfinite(glo) else 0.0
    has_p = np.isfinite(rng["point"][0])
    has_f = np.isfinite(rng["field"][0])
    norm = NormalizationRecord(False) if not enabled else NormalizationRecord(
        True, rng["point"][0] if has_p else None, rng["point"][1] if has_p else None,
        rng["field"][0] if has_f else None, rng["field"][1] if has_f else None)
    # field box over the whole grid and all timesteps + point min/max over all ranks
    inf = float("inf")
    los, his = [], []
    tlo, thi = (float(fld.times.amin()), float(fld.times.amax())) if fld.nt else (inf, -inf)
    tlo, thi = global_minmax(tlo, thi, group, dev)
    dims = np.array(grid_dims if grid_dims is not None else fld.dims)
    if np.isfinite(tlo):
        los.append(np.concatenate([fld.origin, [tlo]]))
        his.append(np.concatenate([fld.origin + dims * fld.spacing, [thi]]))
    pl, ph = [], []
    for d in range(4):
        col = pts.xyz[:, d] if d < 3 else pts.t
        lo, hi, bad = _value_range(col)
        if global_sum_int(bad, group, dev):
            raise ValueError("non-finite (NaN or inf) point coordinate")
        lo, hi = global_minmax(lo, hi, group, dev)
        pl.append(lo)
        ph.append(hi)
    if np.all(np.isfinite(pl)):
        los.append(np.array(pl))
        his.append(np.array(ph))
    if not los:
        raise ValueError("no samples of either kind")
    lo = np.min(los, axis=0)
    hi = np.max(his, axis=0)
    span = hi - lo
    hi = np.where(span <= 0, hi + np.maximum(pad, np.abs(hi) * pad) + pad, hi)
    extent = DomainExtent(lo[0], hi[0], lo[1], hi[1], lo[2], hi[2], lo[3], hi[3])
    # the 128-bit sums of all ranks together must not overflow (csrc/run.cu check_ranges
    # bounds each rank's own share)
    n_p = global_sum_int(pts.n, group, dev)
    n_f = global_sum_int(fld.values.numel(), group, dev)
    cmax = float(np.max(np.abs(np.concatenate([lo, hi]))))
    lim = 2.0 ** 62
    if cmax * (n_p + n_f) >= lim or vmax["point"] * n_p >= lim or vmax["field"] * n_f >= lim:
        raise ValueError("sample coordinates or values too large for the exact 128-bit cluster "
                         "sums over all ranks (max |x| * samples must stay below 2^62)")
    return extent, norm


# ============================================================== sharded run


def shard_run_device(pts: DevicePoints, fld: DeviceField, extent: DomainExtent, params,
                     group=None, progress=None, workspace: Optional[torch.Tensor] = None,
                     out: Optional[dict] = None):
    """engine.run over this rank's slab with the per-pass exact exchange."""
    lib = N.load()
    dev = fld.values.device if fld.values.numel() else pts.t.device
    from .engine import make_params
    from .model import interval_distances
    prm = make_params(extent.mins, interval_distances(extent, params.k), params)
    fs, ps = fld.struct(), pts.struct()
    ws_bytes = lib.mfseg_run_workspace_size(C.byref(prm), C.byref(fs), C.byref(ps))
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    base = workspace.data_ptr()

    def reduce_cb(_user, limbs_ptr, n_words, _stream):
        try:
            off = int(limbs_ptr) - base
            view = workspace[off:off + 8 * int(n_words)].view(torch.int64)
            allreduce_limbs(view, group)
            return 0
        except Exception:   # reported by the native loop as a failed reduce
            return 1

    return run_device(pts, fld, extent, params, progress=progress, reduce=reduce_cb,
                      workspace=workspace, out=out)


def segment_sharded(points, fields, params, group=None, field_offset=(0, 0, 0), grid_dims=None,
                    progress=None):
    """pipeline.segment across ranks (pipeline.py:24-45).  `points` / `fields`
    are this rank's share: whole t-bins of timesteps (time slabs) or whole
    z-bins of planes (spatial slabs; `field_offset` = the global index of the
    slab's first cell, `grid_dims` = the whole grid's dims) and the point samples
    in them (see `shard_dataset`).  Upload -> global normalisation and extent ->
    sharded run -> this rank's labels and the (replicated) centre table.

    Returns (Segmentation, NormalizationRecord, per-iteration wall times), like
    pipeline.segment."""
    from .engine import device, field_to_device, points_to_device
    from .pipeline import to_segmentation
    dev = device()
    pts = points_to_device(points, dev)
    fld = field_to_device(fields, dev)
    fld.offset = tuple(int(o) for o in field_offset)
    extent, norm = normalize_and_extent_sharded(pts, fld, params.normalize, group, grid_dims)
    iter_times = []
    last = [time.perf_counter()]

    def sink(it, delta):
        now = time.perf_counter()
        iter_times.append(now - last[0])
        last[0] = now
        if progress is not None:
            progress(it, delta)

    r = shard_run_device(pts, fld, extent, params, group=group, progress=sink)
    return to_segmentation(r, params, extent), norm, iter_times


def host_extent(points, fields, pad: float = 1e-9) -> DomainExtent:
    """ingest.domain_extent (ingest.py:204-227) on host arrays."""
    los, his = [], []
    if fields is not None and len(fields.times) > 0:
        los.append(np.concatenate([fields.origin, [fields.times[0]]]))
        his.append(np.concatenate([np.asarray(fields.origin) + np.array(fields.dims) *
                                   np.asarray(fields.spacing), [fields.times[-1]]]))
    if points is not None and len(points) > 0:
        loc = np.column_stack([points.xyz, points.t])
        los.append(loc.min(axis=0))
        his.append(loc.max(axis=0))
    if not los:
        raise ValueError("no samples: cannot derive a domain extent")
    lo = np.min(los, axis=0)
    hi = np.max(his, axis=0)
    span = hi - lo
    hi = np.where(span <= 0, hi + np.maximum(pad, np.abs(hi) * pad) + pad, hi)
    return DomainExtent(lo[0], hi[0], lo[1], hi[1], lo[2], hi[2], lo[3], hi[3])


def shard_dataset(points, fields, k, rank: int, world: int, axis: str = "t"):
    """This rank's share of a dataset every rank holds on the host: whole bins of
    timesteps (axis "t") or z-planes (axis "z") of the field and the point
    samples whose bin along that axis the rank owns.  The bins come from the
    dataset's own extent and k (engine.py:111-113, model.py:275-280).

    Returns (points, fields, field_offset, grid_dims, point_index, timestep_offset)
    with point_index = the selected rows' indices in the full point set and
    timestep_offset = the global index of the slab's first timestep."""
    from .model import FieldSet, PointSet, interval_distances
    ext = host_extent(points, fields)
    Cs = interval_distances(ext, k)
    mins = ext.mins
    d = 3 if axis == "t" else 2
    if axis == "t":
        coords = np.asarray(fields.times, dtype=np.float64)
    elif axis == "z":
        coords = cell_centres(fields.dims[2], fields.origin[2], fields.spacing[2])
    else:
        raise ValueError("axis must be 't' or 'z'")
    slabs = bin_slabs(coords, mins[d], Cs[d], k[d], world)
    i0, i1 = slabs[rank]
    b0, b1 = slab_bin_ranges(coords, mins[d], Cs[d], k[d], slabs)[rank]
    nx, ny, nz = fields.dims
    vals = np.asarray(fields.values).reshape(len(fields.times), nz, ny * nx)
    if axis == "t":
        fs = FieldSet(tuple(fields.dims), fields.origin, fields.spacing,
                      np.asarray(fields.times)[i0:i1], vals[i0:i1].reshape(i1 - i0, -1))
        off, m0 = (0, 0, 0), i0
    else:
        fs = FieldSet((nx, ny, i1 - i0), fields.origin, fields.spacing, fields.times,
                      np.ascontiguousarray(vals[:, i0:i1]).reshape(len(fields.times), -1))
        off, m0 = (0, 0, i0), 0
    if points is not None and len(points) > 0:
        col = np.asarray(points.t) if axis == "t" else np.asarray(points.xyz)[:, 2]
        idx = np.flatnonzero(select_points_for_slab(col, mins[d], Cs[d], k[d], b0, b1))
        ps = PointSet(np.asarray(points.traj_id)[idx], np.asarray(points.t)[idx],
                      np.asarray(points.xyz)[idx], np.asarray(points.value)[idx])
    else:
        idx = np.zeros(0, np.int64)
        ps = points
    return ps, fs, off, tuple(fields.dims), idx, m0
