"""Multi-GPU segmentation: time slabs across ranks, one exact exchange per pass.

The reference is single-process; the paper sketches
per-iteration centre merging across GPUs as future work.
Here every rank owns a contiguous slab of field timesteps and the point samples
whose t falls in it.  Labels are independent given the (replicated) centres,
so the only data-path collective is, once per pass, a SUM all-reduce of the
per-cluster partial sums.  Those sums are 128-bit fixed-point integers
(exact), exchanged as three 42-bit limbs per word, so the reduced sums and
therefore the centres and labels are bit-identical for any number of ranks.

Host-side pieces (slab split, min/max and extent agreement, the limb
all-reduce) are plain torch.distributed and are exercised on CPU with gloo
by tests/test_parallel.py.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .engine import DeviceField, DevicePoints, run_device, stream_ptr
from .model import DomainExtent


def time_slab(rank: int, world: int, nt: int):
    """[m0, m1) timestep range of `rank` (contiguous, sizes differ by <= 1)."""
    base, extra = divmod(nt, world)
    m0 = rank * base + min(rank, extra)
    return m0, m0 + base + (1 if rank < extra else 0)


def tbin_slabs(times, t_min: float, C_t: float, k_t: int, world: int):
    """Contiguous timestep slabs [m0, m1) per rank whose boundaries fall on t-bin
    changes (bin = clip(floor((t - t_min) / C_t), 0, k_t - 1), engine.py:111-113),
    as balanced as the bin boundaries allow.  Whole t-bins per rank keep every
    field and point tile on one GPU, so the fixed-order partial sums (and the
    centres) are bit-identical for any rank count."""
    t = np.asarray(times, dtype=np.float64)
    nt = len(t)
    b = np.clip(np.floor((t - t_min) / C_t), 0, k_t - 1).astype(np.int64)
    cuts = np.flatnonzero(b[1:] != b[:-1]) + 1          # allowed slab starts
    bounds = [0]
    for r in range(1, world):
        target = r * nt / world
        ok = cuts[cuts >= bounds[-1]]
        bounds.append(int(ok[np.argmin(np.abs(ok - target))]) if len(ok) else nt)
    bounds.append(nt)
    return [(bounds[r], max(bounds[r], bounds[r + 1])) for r in range(world)]


def global_minmax(lo: float, hi: float, group=None, device=None):
    """Exact global (min, max) of per-rank values (inf/-inf for empty ranks)."""
    t = torch.tensor([lo, -hi], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return float(t[0]), float(-t[1])


def allreduce_limbs(limbs: torch.Tensor, group=None) -> None:
    """In-place SUM of int64 limb words across ranks (exact: each limb < 2^42)."""
    dist.all_reduce(limbs, op=dist.ReduceOp.SUM, group=group)


def normalize_and_extent_sharded(pts: DevicePoints, fld: DeviceField, t_range=None, group=None,
                                 pad: float = 1e-9) -> DomainExtent:
    """normalize_variables + domain_extent over the union of all ranks' slabs
    (ingest.py:204-227, 312-335), identical to the single-GPU result."""
    lib = N.load()
    dev = fld.values.device
    inf = float("inf")
    for vals in (pts.value, fld.values):
        lo = float(vals.amin()) if vals.numel() else inf
        hi = float(vals.amax()) if vals.numel() else -inf
        glo, ghi = global_minmax(lo, hi, group, dev)
        if vals.numel() and np.isfinite(glo):
            N.check(lib.mfseg_normalize_range(N.ptr(vals), vals.numel(), glo, ghi, stream_ptr()),
                    "mfseg_normalize_range")
    # field box over all timesteps + point min/max over all ranks
    los, his = [], []
    tlo = float(fld.times.amin()) if fld.nt else inf
    thi = float(fld.times.amax()) if fld.nt else -inf
    tlo, thi = global_minmax(tlo, thi, group, dev)
    if np.isfinite(tlo):
        los.append(np.concatenate([fld.origin, [tlo]]))
        his.append(np.concatenate([fld.origin + np.array(fld.dims) * fld.spacing, [thi]]))
    pl, ph = [], []
    for d in range(4):
        col = pts.xyz[:, d] if d < 3 else pts.t
        lo = float(col.amin()) if pts.n else inf
        hi = float(col.amax()) if pts.n else -inf
        lo, hi = global_minmax(lo, hi, group, dev)
        pl.append(lo)
        ph.append(hi)
    if np.all(np.isfinite(pl)):
        los.append(np.array(pl))
        his.append(np.array(ph))
    lo = np.min(los, axis=0)
    hi = np.max(his, axis=0)
    span = hi - lo
    hi = np.where(span <= 0, hi + np.maximum(pad, np.abs(hi) * pad) + pad, hi)
    return DomainExtent(lo[0], hi[0], lo[1], hi[1], lo[2], hi[2], lo[3], hi[3])


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


def segment_sharded(points, fields, params, group=None):
    """pipeline.segment across ranks: this rank's host slab (whole t-bins of the
    field timesteps and the points in them, see tbin_slabs) -> upload ->
    global normalisation and extent -> sharded run -> this rank's labels and the
    (replicated) centre table.  Returns (Segmentation, extent)."""
    from .engine import device, field_to_device, points_to_device
    from .pipeline import to_segmentation
    dev = device()
    pts = points_to_device(points, dev)
    fld = field_to_device(fields, dev)
    extent = normalize_and_extent_sharded(pts, fld, group=group)
    r = shard_run_device(pts, fld, extent, params, group=group)
    return to_segmentation(r, params, extent), extent
