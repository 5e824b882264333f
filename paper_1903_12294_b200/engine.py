"""GPU-backed drop-in for the reference's `mfseg.engine` (engine.py:1-396).

Same function names, signatures, return types and errors.  Every data-parallel
step runs in libmfseg_sm100.so on the current CUDA device:

  run                 -> mfseg_run      (seed, CenterGrid, assign, accumulate,
                                         update, converge: one native loop)
  assign_iteration    -> mfseg_assign   (windowed exact-fp64 argmin)
  accumulate          -> mfseg_accumulate (exact 128-bit fixed-point sums)
  update_centers      -> mfseg_update_centers_f64
  has_converged /
  max_center_delta    -> mfseg_compare_centers

`workers` and `chunk_size` are accepted for signature compatibility; like the
reference's, the results do not depend on them (engine.py:9-12).

Numerical contract: labels are bit-identical to the reference for the same
centres (exact predicate, reference operation order, no FMA).  Centre sums
are exact (correctly rounded once) instead of numpy's sequential order, so
centres agree to ~1e-15 relative; with dyadic inputs every sum is exact in
both and the whole run is bit-identical.
"""

from __future__ import annotations

import gc
import threading

import ctypes as C
import itertools
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import _native as N
from .model import (ClusterCenter, ClusterParams, DomainExtent, FieldSet, PointSet,
                    Segmentation, interval_distances, space_time_distance)

ProgressSink = Callable[[int, float], None]


# ============================================================== device helpers

def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the sm_100a segmentation path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


class _Stager:
    """Pageable host -> device uploads through a ring of pinned staging buffers:
    host threads fill the slots (torch's copy releases the GIL) while the copy
    engine drains the filled ones, so a pageable array moves at several times the
    rate of a direct pageable copy (which the driver stages through one small
    buffer synchronously).  One per process, serialised by a lock."""

    SLOT = 32 << 20
    SLOTS = 8

    def __init__(self):
        self.lock = threading.Lock()
        self.ring = None
        self.pool = None

    def _init(self):
        if self.ring is None:
            from concurrent.futures import ThreadPoolExecutor
            self.ring = [torch.empty(self.SLOT, dtype=torch.uint8, pin_memory=True)
                         for _ in range(self.SLOTS)]
            self.pool = ThreadPoolExecutor(self.SLOTS, thread_name_prefix="mfseg-stage")

    def upload(self, src: torch.Tensor, dst: torch.Tensor) -> None:
        """dst (device, contiguous) <- src (host, contiguous, same bytes), ordered
        on the current stream; returns once the last slot is queued."""
        with self.lock:
            self._init()
            sb = src.reshape(-1).view(torch.uint8)
            db = dst.reshape(-1).view(torch.uint8)
            n = sb.numel()
            nch = -(-n // self.SLOT)
            stream = torch.cuda.current_stream()
            events = [None] * self.SLOTS
            futs = {}

            def fill(i):
                a = i * self.SLOT
                b = min(n, a + self.SLOT)
                self.ring[i % self.SLOTS][:b - a].copy_(sb[a:b])
                return a, b

            for i in range(min(self.SLOTS, nch)):
                futs[i] = self.pool.submit(fill, i)
            for i in range(nch):
                a, b = futs.pop(i).result()
                slot = i % self.SLOTS
                db[a:b].copy_(self.ring[slot][:b - a], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                events[slot] = ev
                j = i + self.SLOTS
                if j < nch:
                    ev.synchronize()          # the slot's DMA is done: refill it
                    futs[j] = self.pool.submit(fill, j)
            for ev in events:
                if ev is not None:
                    ev.synchronize()          # ring buffers are reused by the next call

    def download(self, src: torch.Tensor, dst: torch.Tensor) -> None:
        """dst (host, pageable, contiguous) <- src (device, contiguous, same bytes):
        the copy engine fills the pinned slots in turn on the current stream and
        host threads drain each into dst once its DMA has completed."""
        with self.lock:
            self._init()
            sb = src.reshape(-1).view(torch.uint8)
            db = dst.reshape(-1).view(torch.uint8)
            n = sb.numel()
            nch = -(-n // self.SLOT)
            stream = torch.cuda.current_stream()
            drains = [None] * self.SLOTS

            def drain(slot, a, b, ev):
                ev.synchronize()
                db[a:b].copy_(self.ring[slot][:b - a])

            for i in range(nch):
                slot = i % self.SLOTS
                if drains[slot] is not None:
                    drains[slot].result()      # the slot's previous chunk is out
                a = i * self.SLOT
                b = min(n, a + self.SLOT)
                self.ring[slot][:b - a].copy_(sb[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                drains[slot] = self.pool.submit(drain, slot, a, b, ev)
            for f in drains:
                if f is not None:
                    f.result()


_stager = _Stager()
_STAGE_MIN_BYTES = 16 << 20


def upload(t: torch.Tensor, dev=None) -> torch.Tensor:
    """Host tensor -> device tensor of the same dtype on the current stream:
    pinned memory by direct DMA (asynchronous), large pageable arrays through
    the pinned staging ring, small ones by a plain copy."""
    dev = dev or device()
    t = t.contiguous()
    if t.device.type == "cuda":
        return t.to(dev)
    nbytes = t.numel() * t.element_size()
    if nbytes < _STAGE_MIN_BYTES or t.is_pinned():
        return t.to(device=dev, non_blocking=True)
    out = torch.empty(t.shape, dtype=t.dtype, device=dev)
    _stager.upload(t, out)
    return out


def to_dev(a, dtype=torch.float64, dev=None):
    """Host array (numpy / tensor) -> contiguous device tensor of `dtype`.  The
    bytes cross PCIe in the array's own dtype (e.g. f32 field values) and are
    converted on the device (f32 -> f64 widening is exact, as the reference's
    host-side astype, ingest.py:39-78); see `upload` for pinned / pageable."""
    dev = dev or device()
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(a))
    d = upload(t, dev)
    return d if d.dtype == dtype else d.to(dtype)


def to_host_async(t: torch.Tensor):
    """Start a device -> pinned host copy; returns (host tensor, event).  The
    numpy view is valid once the event has completed (see `host_ready`)."""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    if t.numel():
        h.copy_(t, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    return h, ev


def host_ready(pending) -> np.ndarray:
    h, ev = pending
    ev.synchronize()
    return h.numpy()


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy through a pinned staging buffer (fast D2H DMA)."""
    if t.numel() == 0:
        return t.cpu().numpy()
    return host_ready(to_host_async(t))


def download(t: torch.Tensor, dtype=None) -> np.ndarray:
    """Device tensor -> new pageable numpy array (converted to `dtype` on the
    device first, e.g. int32 -> int64 indices): large arrays through the pinned
    staging ring, without allocating page-locked memory of their size."""
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    t = t.contiguous()
    nbytes = t.numel() * t.element_size()
    if t.device.type != "cuda" or nbytes < _STAGE_MIN_BYTES:
        return t.cpu().numpy()
    out = torch.empty(t.shape, dtype=t.dtype)
    _stager.download(t, out)
    return out.numpy()


@dataclass
class DeviceField:
    dims: tuple
    origin: np.ndarray
    spacing: np.ndarray
    times: torch.Tensor      # (T,) f64
    values: torch.Tensor     # (T * ncell,) f64
    offset: tuple = (0, 0, 0)   # global cell index of the first cell (spatial slabs)

    @property
    def nt(self):
        return int(self.times.numel())

    def struct(self) -> N.Field:
        f = N.Field()
        if self.nt == 0:
            f.nx = f.ny = f.nz = 1
            f.nt = 0
            return f
        f.nx, f.ny, f.nz = (int(d) for d in self.dims)
        f.nt = self.nt
        for d in range(3):
            f.origin[d] = float(self.origin[d])
            f.spacing[d] = float(self.spacing[d])
        f.times = N.ptr(self.times)
        f.values = N.ptr(self.values)
        for d in range(3):
            f.offset[d] = int(self.offset[d])
        return f


@dataclass
class DevicePoints:
    xyz: torch.Tensor        # (N, 3) f64
    t: torch.Tensor          # (N,)
    value: torch.Tensor      # (N,)

    @property
    def n(self):
        return int(self.t.numel())

    def struct(self) -> N.Points:
        p = N.Points()
        p.n = self.n
        if self.n:
            p.xyz, p.t, p.value = N.ptr(self.xyz), N.ptr(self.t), N.ptr(self.value)
        return p


def field_to_device(fields, dev=None) -> DeviceField:
    if fields is None or len(fields) == 0:
        dev = dev or device()
        return DeviceField((1, 1, 1), np.zeros(3), np.ones(3),
                           torch.zeros(0, dtype=torch.float64, device=dev),
                           torch.zeros(0, dtype=torch.float64, device=dev))
    return DeviceField(tuple(int(d) for d in fields.dims), np.asarray(fields.origin, float),
                       np.asarray(fields.spacing, float), to_dev(fields.times, dev=dev),
                       to_dev(np.asarray(fields.values).reshape(-1), dev=dev))


def points_to_device(points, dev=None) -> DevicePoints:
    dev = dev or device()
    if points is None or len(points) == 0:
        z = torch.zeros(0, dtype=torch.float64, device=dev)
        return DevicePoints(z.reshape(0, 3), z, z)
    return DevicePoints(to_dev(np.asarray(points.xyz).reshape(-1, 3), dev=dev),
                        to_dev(points.t, dev=dev), to_dev(points.value, dev=dev))


def make_params(mins, C, params, w=None) -> N.Params:
    """Fill the ABI params; `w` overrides (w_d, w_p, w_f)."""
    p = N.Params()
    for d in range(4):
        p.k[d] = int(params.k[d])
        p.mins[d] = float(mins[d])
        p.C[d] = float(C[d])
    p.c_f = float(params.c_f)
    p.w_d, p.w_p, p.w_f = (float(params.w_d), float(params.w_p), float(params.w_f)) if w is None else w
    p.eps_c = float(params.eps_c)
    p.max_iterations = int(getattr(params, "max_iterations", 50))
    return p


# ============================================================== centre state

def seed_centers(extent: DomainExtent, k) -> np.ndarray:
    """(K, 4) seeds at the k-grid cell midpoints, ids t-major then z, y, x
    (engine.py:31-45).  O(K) host helper; `run` seeds on the device."""
    C = interval_distances(extent, k)
    mins = extent.mins
    ax = [mins[d] + (np.arange(k[d]) + 0.5) * C[d] for d in range(4)]
    grid = np.meshgrid(ax[3], ax[2], ax[1], ax[0], indexing="ij")
    return np.column_stack([grid[3].ravel(), grid[2].ravel(), grid[1].ravel(), grid[0].ravel()])


@dataclass
class CenterState:
    """Per-id centre arrays (engine.py:48-86); host numpy mirror of the device state."""

    loc: np.ndarray
    pval: np.ndarray
    fval: np.ndarray
    has_p: np.ndarray
    has_f: np.ndarray
    n_points: np.ndarray
    n_fields: np.ndarray
    dormant: np.ndarray

    @classmethod
    def from_seeds(cls, seeds: np.ndarray) -> "CenterState":
        K = len(seeds)
        return cls(np.array(seeds, dtype=float, copy=True), np.full(K, np.nan), np.full(K, np.nan),
                   np.zeros(K, bool), np.zeros(K, bool), np.zeros(K, np.int64),
                   np.zeros(K, np.int64), np.zeros(K, bool))

    def to_table(self) -> list:
        """Live clusters only, as the public centre table (engine.py:72-86)."""
        live = np.flatnonzero(self.n_points + self.n_fields > 0)
        loc = self.loc[live].tolist()
        pv = np.where(self.has_p[live], self.pval[live], np.nan).tolist()
        fv = np.where(self.has_f[live], self.fval[live], np.nan).tolist()
        hp, hf = self.has_p[live].tolist(), self.has_f[live].tolist()
        npt, nfl = self.n_points[live].tolist(), self.n_fields[live].tolist()
        # tens of thousands of small objects: keep the cyclic GC from rescanning
        # the heap several times while they are created (none of them is cyclic)
        gc_on = gc.isenabled()
        gc.disable()
        try:
            return [ClusterCenter(c, l[0], l[1], l[2], l[3], p if a else None, f if b else None,
                                  n1, n2)
                    for c, l, p, f, a, b, n1, n2 in zip(live.tolist(), loc, pv, fv, hp, hf, npt, nfl)]
        finally:
            if gc_on:
                gc.enable()

    # --- device round trip -------------------------------------------------
    def to_device(self, dev=None) -> dict:
        dev = dev or device()
        return {
            "loc": to_dev(np.asarray(self.loc, float).T.copy(), dev=dev),   # (4, K) planes
            "pval": to_dev(self.pval, dev=dev), "fval": to_dev(self.fval, dev=dev),
            "has_p": to_dev(np.asarray(self.has_p, np.uint8), torch.uint8, dev),
            "has_f": to_dev(np.asarray(self.has_f, np.uint8), torch.uint8, dev),
            "dormant": to_dev(np.asarray(self.dormant, np.uint8), torch.uint8, dev),
            "n_points": to_dev(np.asarray(self.n_points, np.int64), torch.int64, dev),
            "n_fields": to_dev(np.asarray(self.n_fields, np.int64), torch.int64, dev),
        }

    @classmethod
    def from_device(cls, d: dict) -> "CenterState":
        # one packed D2H copy instead of eight
        K = d["pval"].numel()
        f = torch.cat([d["loc"].reshape(-1), d["pval"], d["fval"],
                       d["n_points"].view(torch.float64), d["n_fields"].view(torch.float64)])
        b = torch.cat([d["has_p"], d["has_f"], d["dormant"]])
        fh, bh = to_host(f), to_host(b).astype(bool)
        ints = fh[6 * K:].view(np.int64)
        return cls(fh[:4 * K].reshape(4, K).T.copy(), fh[4 * K:5 * K].copy(),
                   fh[5 * K:6 * K].copy(), bh[:K], bh[K:2 * K], ints[:K].copy(),
                   ints[K:].copy(), bh[2 * K:])


def empty_state(K: int, dev=None) -> dict:
    dev = dev or device()
    f = dict(dtype=torch.float64, device=dev)
    return {"loc": torch.empty((4, K), **f), "pval": torch.empty(K, **f),
            "fval": torch.empty(K, **f),
            "has_p": torch.empty(K, dtype=torch.uint8, device=dev),
            "has_f": torch.empty(K, dtype=torch.uint8, device=dev),
            "dormant": torch.empty(K, dtype=torch.uint8, device=dev),
            "n_points": torch.empty(K, dtype=torch.int64, device=dev),
            "n_fields": torch.empty(K, dtype=torch.int64, device=dev)}


def state_struct(d: dict) -> N.Centers:
    c = N.Centers()
    for name in ("loc", "pval", "fval", "has_p", "has_f", "dormant", "n_points", "n_fields"):
        setattr(c, name, N.ptr(d[name]))
    return c


class CenterGrid:
    """engine.CenterGrid (engine.py:89-134).  Holds the binning geometry; the
    device rebuilds the bin CSR and neighbour lists from the centre locations
    on every pass.  `candidates` / `sample_bins` are O(K) host inspection
    helpers with the reference's semantics."""

    _OFFSETS = np.array(list(itertools.product((-1, 0, 1), repeat=4)))

    def __init__(self, loc: np.ndarray, extent: DomainExtent, C: np.ndarray, k):
        self.loc = np.asarray(loc, float)
        self.C = np.asarray(C, float)
        self.mins = extent.mins
        self.k = np.asarray(k)

    def _bin_indices(self, loc):
        return np.clip(np.floor((loc - self.mins) / self.C).astype(np.int64), 0, self.k - 1)

    def _flatten(self, idx):
        kx, ky, kz, _ = self.k
        return ((idx[..., 3] * kz + idx[..., 2]) * ky + idx[..., 1]) * kx + idx[..., 0]

    def sample_bins(self, loc):
        return self._bin_indices(loc)

    def candidates(self, bin4) -> np.ndarray:
        cb = self._bin_indices(self.loc)
        near = np.all(np.abs(cb - np.asarray(bin4)) <= 1, axis=1)
        return np.flatnonzero(near)


# ============================================================== metrics (scalar helpers)

def point_distance(loc4, value: float, center: ClusterCenter, params: ClusterParams) -> float:
    """w_p |p_s - p_c| + w_d S_st (engine.py:152-155)."""
    vt = params.w_p * abs(value - center.p_c) if center.p_c is not None else 0.0
    return float(vt + params.w_d * space_time_distance(loc4, center.loc4, params.c_f))


def field_distance(loc4, value: float, center: ClusterCenter, params: ClusterParams) -> float:
    """w_f |f_s - f_c| + w_d S_st (engine.py:158-161)."""
    vt = params.w_f * abs(value - center.f_c) if center.f_c is not None else 0.0
    return float(vt + params.w_d * space_time_distance(loc4, center.loc4, params.c_f))


# ============================================================== assignment

def _run_assign(pts: DevicePoints, fld: DeviceField, state: dict, prm: N.Params, K: int):
    lib = N.load()
    dev = state["loc"].device
    prm.n_centers = K
    fs, ps = fld.struct(), pts.struct()
    ws_bytes = lib.mfseg_assign_workspace_size(C.byref(prm), C.byref(fs), C.byref(ps))
    if ws_bytes == 0:
        N.check(2, "mfseg_assign_workspace_size")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    pl = torch.empty(pts.n, dtype=torch.int32, device=dev)
    fl = torch.empty(fld.values.numel(), dtype=torch.int32, device=dev)
    acc = torch.empty((K, N.ACC_WORDS), dtype=torch.int64, device=dev)
    N.check(lib.mfseg_assign(C.byref(prm), C.byref(fs), C.byref(ps), state_struct(state),
                             N.ptr(pl) if pts.n else None, N.ptr(fl) if fld.nt else None,
                             N.ptr(acc), N.ptr(ws), ws_bytes, stream_ptr()), "mfseg_assign")
    return pl, fl, acc


def assign_iteration(points: PointSet, fields: FieldSet, field_loc4, centers: CenterState,
                     grid: CenterGrid, params: ClusterParams, C: np.ndarray,
                     workers: int = 1, chunk_size: Optional[int] = None):
    """Assign all samples of both kinds; returns (point_labels, field_labels)
    as int64 numpy arrays (engine.py:208-218).  `field_loc4` is not read: field
    locations are re-derived from the grid indices on the device."""
    dev = device()
    K = len(centers.loc)
    prm = make_params(grid.mins, C, params)
    pl, fl, _ = _run_assign(points_to_device(points, dev), field_to_device(fields, dev),
                            centers.to_device(dev), prm, K)
    return pl.cpu().numpy().astype(np.int64), fl.cpu().numpy().astype(np.int64)


def acc_to_numpy(acc: torch.Tensor, K: int):
    """128-bit accumulators -> (sums (K,4), psum, fsum, n_p, n_f) like accumulate()."""
    lib = N.load()
    dev = acc.device
    sums = torch.empty((K, 4), dtype=torch.float64, device=dev)
    psum = torch.empty(K, dtype=torch.float64, device=dev)
    fsum = torch.empty(K, dtype=torch.float64, device=dev)
    n_p = torch.empty(K, dtype=torch.int64, device=dev)
    n_f = torch.empty(K, dtype=torch.int64, device=dev)
    N.check(lib.mfseg_acc_to_double(K, N.ptr(acc), N.ptr(sums), N.ptr(psum), N.ptr(fsum),
                                    N.ptr(n_p), N.ptr(n_f), stream_ptr()), "mfseg_acc_to_double")
    return (sums.cpu().numpy(), psum.cpu().numpy(), fsum.cpu().numpy(), n_p.cpu().numpy(),
            n_f.cpu().numpy())


def accumulate(point_labels, points: PointSet, field_labels, fields: FieldSet, field_loc4,
               K: int):
    """Per-cluster sums over the full label arrays (engine.py:244-263), exact."""
    lib = N.load()
    dev = device()
    pts = points_to_device(points, dev)
    fld = field_to_device(fields, dev)
    pl = to_dev(np.asarray(point_labels, np.int64), torch.int32, dev) if pts.n else None
    fl = to_dev(np.asarray(field_labels, np.int64), torch.int32, dev) if fld.nt else None
    for lab in (pl, fl):
        if lab is not None and lab.numel() and (int(lab.min()) < 0 or int(lab.max()) >= K):
            raise ValueError("labels must lie in [0, K)")
    acc = torch.empty((K, N.ACC_WORDS), dtype=torch.int64, device=dev)
    fs, ps = fld.struct(), pts.struct()
    N.check(lib.mfseg_accumulate(K, C.byref(fs), C.byref(ps), N.ptr(pl), N.ptr(fl), N.ptr(acc),
                                 stream_ptr()), "mfseg_accumulate")
    return acc_to_numpy(acc, K)


def update_centers(centers: CenterState, sums, psum, fsum, n_p, n_f) -> CenterState:
    """Member means; empty clusters freeze and go dormant (engine.py:266-286)."""
    lib = N.load()
    dev = device()
    K = len(centers.loc)
    old = centers.to_device(dev)
    new = empty_state(K, dev)
    # keep every uploaded tensor referenced until the kernel has consumed it
    args = (to_dev(np.asarray(sums, float).reshape(K, 4), dev=dev), to_dev(psum, dev=dev),
            to_dev(fsum, dev=dev), to_dev(np.asarray(n_p, np.int64), torch.int64, dev),
            to_dev(np.asarray(n_f, np.int64), torch.int64, dev))
    N.check(lib.mfseg_update_centers_f64(K, *(N.ptr(a) for a in args), state_struct(old),
                                         state_struct(new), stream_ptr()),
            "mfseg_update_centers_f64")
    return CenterState.from_device(new)


def _compare(old: CenterState, new: CenterState, eps_c: float):
    lib = N.load()
    dev = device()
    conv, delta = C.c_int32(0), C.c_double(0.0)
    a, b = old.to_device(dev), new.to_device(dev)
    N.check(lib.mfseg_compare_centers(len(old.loc), state_struct(a), state_struct(b),
                                      float(eps_c), C.byref(conv), C.byref(delta), stream_ptr()),
            "mfseg_compare_centers")
    return bool(conv.value), float(delta.value)


def has_converged(old: CenterState, new: CenterState, eps_c: float) -> bool:
    """engine.py:293-307."""
    return _compare(old, new, eps_c)[0]


def max_center_delta(old: CenterState, new: CenterState) -> float:
    """engine.py:310-320."""
    return _compare(old, new, 1.0)[1]


# ============================================================== full run

@dataclass
class DeviceRun:
    """Result of run_device: device tensors + loop outcome."""

    point_labels: torch.Tensor   # int32 (N_p,), record order
    field_labels: torch.Tensor   # int32 (N_f,), timestep-major x-fastest
    state: dict                  # final centre state (device tensors)
    iterations_used: int
    converged: bool


def _check_run_inputs(n_points: int, n_fields: int, params) -> None:
    # engine.py:331-338
    if n_points == 0 and n_fields == 0:
        raise ValueError("no samples of either kind")
    if n_points > 0 and params.w_d + params.w_p <= 0:
        raise ValueError("point metric is identically zero")
    if n_fields > 0 and params.w_d + params.w_f <= 0:
        raise ValueError("field metric is identically zero")


def run_device(pts: DevicePoints, fld: DeviceField, extent: DomainExtent, params,
               progress: Optional[ProgressSink] = None, reduce=None,
               workspace: Optional[torch.Tensor] = None,
               out: Optional[dict] = None) -> DeviceRun:
    """engine.run on device-resident inputs (normalized values)."""
    _check_run_inputs(pts.n, int(fld.values.numel()), params)
    lib = N.load()
    dev = fld.values.device if fld.values.numel() else pts.t.device
    C_ = interval_distances(extent, params.k)
    prm = make_params(extent.mins, C_, params)
    K = int(np.prod(params.k))
    fs, ps = fld.struct(), pts.struct()
    ws_bytes = lib.mfseg_run_workspace_size(C.byref(prm), C.byref(fs), C.byref(ps))
    if ws_bytes == 0:
        N.check(2, "mfseg_run_workspace_size")
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    if out is None:
        out = {"point_labels": torch.empty(pts.n, dtype=torch.int32, device=dev),
               "field_labels": torch.empty(fld.values.numel(), dtype=torch.int32, device=dev),
               "state": empty_state(K, dev)}
    errors = []

    def _prog(_user, it, delta):
        if progress is not None and not errors:
            try:
                progress(int(it), float(delta))
            except BaseException as e:   # re-raised after the native loop returns
                errors.append(e)

    cb = N.PROGRESS_FN(_prog)
    rcb = N.REDUCE_FN(reduce) if reduce is not None else N.REDUCE_FN()
    it, conv = C.c_int32(0), C.c_int32(0)
    N.check(lib.mfseg_run(C.byref(prm), C.byref(fs), C.byref(ps),
                          N.ptr(out["point_labels"]) if pts.n else None,
                          N.ptr(out["field_labels"]) if fld.nt else None,
                          state_struct(out["state"]), C.byref(it), C.byref(conv), cb, None,
                          rcb, None, N.ptr(workspace), ws_bytes, stream_ptr()), "mfseg_run")
    if errors:
        raise errors[0]
    return DeviceRun(out["point_labels"], out["field_labels"], out["state"], int(it.value),
                     bool(conv.value))


def run(points: Optional[PointSet], fields: Optional[FieldSet], extent: DomainExtent,
        params: ClusterParams, workers: int = 1, chunk_size: Optional[int] = None,
        progress: Optional[ProgressSink] = None) -> Segmentation:
    """Full clustering run: seed, iterate, converge (engine.py:323-381).

    Inputs are host arrays (as in the reference); they are copied to the GPU,
    segmented there, and labels + centre table come back to the host.
    """
    points = points if points is not None else PointSet.empty()
    fields = fields if fields is not None else FieldSet.empty()
    _check_run_inputs(len(points), len(fields), params)
    dev = device()
    r = run_device(points_to_device(points, dev), field_to_device(fields, dev), extent, params,
                   progress=progress)
    state = CenterState.from_device(r.state)
    return Segmentation(point_labels=to_host(r.point_labels),
                        field_labels=to_host(r.field_labels),
                        centers=state.to_table(), params=params, extent=extent,
                        iterations_used=r.iterations_used, converged=r.converged)


def initial_assignment(points: PointSet, fields: FieldSet, extent: DomainExtent,
                       params: ClusterParams, workers: int = 1,
                       chunk_size: Optional[int] = None):
    """Nearest-seed assignment under the space-time metric only (engine.py:384-396)."""
    C_ = interval_distances(extent, params.k)
    cs = CenterState.from_seeds(seed_centers(extent, params.k))
    zero = ClusterParams(k=tuple(params.k), c_f=params.c_f, w_d=1.0, w_p=0.0, w_f=0.0,
                         eps_c=params.eps_c)
    return assign_iteration(points, fields, None, cs, CenterGrid(cs.loc, extent, C_, params.k),
                            zero, C_, workers, chunk_size)
