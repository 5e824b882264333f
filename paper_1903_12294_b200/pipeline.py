"""`pipeline.segment` equivalent (pipeline.py:24-45): normalize -> extent -> run,
with the data uploaded once and every step on the device."""

from __future__ import annotations

import time
from typing import Optional

import numpy as np

from .engine import (CenterState, DeviceField, DevicePoints, DeviceRun, device, field_to_device,
                     points_to_device, run_device, host_ready, to_host_async)
from .ingest import NormalizationRecord, domain_extent_device, normalize_device
from .model import ClusterParams, FieldSet, PointSet, Segmentation


def segment_device(pts: DevicePoints, fld: DeviceField, params: ClusterParams, progress=None,
                   reduce=None, workspace=None, out=None):
    """Normalize (in place), derive the extent and run, all on device tensors.

    Returns (DeviceRun, NormalizationRecord, extent, per-iteration wall times).
    """
    norm = normalize_device(pts, fld, params.normalize)
    extent = domain_extent_device(pts, fld)
    iter_times = []
    last = [time.perf_counter()]

    def sink(it, delta):
        now = time.perf_counter()
        iter_times.append(now - last[0])
        last[0] = now
        if progress is not None:
            progress(it, delta)

    r = run_device(pts, fld, extent, params, progress=sink, reduce=reduce, workspace=workspace,
                   out=out)
    return r, norm, extent, iter_times


def segment(points: Optional[PointSet], fields: Optional[FieldSet], params: ClusterParams,
            workers: int = 1, chunk_size: Optional[int] = None, progress=None):
    """Host arrays in, (Segmentation, NormalizationRecord, iteration wall times) out."""
    dev = device()
    pts = points_to_device(points, dev)
    fld = field_to_device(fields, dev)
    r, norm, extent, iter_times = segment_device(pts, fld, params, progress=progress)
    seg = to_segmentation(r, params, extent)
    return seg, norm, iter_times


def to_segmentation(r: DeviceRun, params, extent) -> Segmentation:
    # label copies run on the copy engine while the host builds the centre table
    state = CenterState.from_device(r.state)
    pl, fl = to_host_async(r.point_labels), to_host_async(r.field_labels)
    table = state.to_table()
    return Segmentation(point_labels=host_ready(pl), field_labels=host_ready(fl), centers=table,
                        params=params, extent=extent, iterations_used=r.iterations_used,
                        converged=r.converged)


def segment_from_files(field_path: str, points: Optional[PointSet], params: ClusterParams,
                       progress=None):
    """pipeline.segment over a field stored in the reference's format
    (ingest.py:39-78): the per-timestep files stream into device memory
    (ingest.load_field_device) instead of materialising a host FieldSet.
    Returns (Segmentation, NormalizationRecord, iteration wall times)."""
    from .ingest import load_field_device
    dev = device()
    fld = load_field_device(field_path, dev)
    pts = points_to_device(points, dev)
    r, norm, extent, iter_times = segment_device(pts, fld, params, progress=progress)
    return to_segmentation(r, params, extent), norm, iter_times


def segment_to_dir(outdir: str, field_path: Optional[str], points: Optional[PointSet],
                   params: ClusterParams, workers: int = 1, chunk_size: Optional[int] = None,
                   progress=None):
    """pipeline.segment_to_dir (pipeline.py:48-70): a run directory from a field
    file in the reference's format (streamed into device memory) and in-memory
    points (the reference's CSV / derivation front end is host I/O, out of scope).

    Labels go from device memory straight to the label files
    (artifacts.save_segmentation_device); report.json carries the reference's
    keys plus throughput keys (`voxel_timesteps_per_s`, `passes`,
    `device_seconds`).  Returns (DeviceRun, NormalizationRecord, extent)."""
    import torch
    from . import artifacts
    from .ingest import load_field_device
    dev = device()
    t0 = time.perf_counter()
    fld = load_field_device(field_path, dev) if field_path else field_to_device(None, dev)
    pts = points_to_device(points, dev)
    t1 = time.perf_counter()
    r, norm, extent, iter_times = segment_device(pts, fld, params, progress=progress)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    artifacts.save_segmentation_device(outdir, r, params, extent, norm)
    n_f = int(r.field_labels.numel())
    passes = 1 + r.iterations_used
    artifacts.save_report(outdir, {
        "inputs": {"field": field_path, "points": None if points is None else "in-memory",
                   "derive": None},
        "params": params.to_dict(),
        "workers": workers,
        "chunk_size": chunk_size,
        "n_point_samples": int(r.point_labels.numel()),
        "n_field_samples": n_f,
        "iterations_used": r.iterations_used,
        "converged": r.converged,
        "iteration_seconds": iter_times,
        "total_seconds": t2 - t1,
        # extra keys (the deterministic artifacts are untouched)
        "device": torch.cuda.get_device_name(dev),
        "passes": passes,
        "device_seconds": t2 - t1,
        "load_seconds": t1 - t0,
        "voxel_timesteps_per_s": n_f / (t2 - t1) if t2 > t1 else None,
    })
    return r, norm, extent
