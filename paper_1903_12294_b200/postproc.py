"""GPU-backed drop-in for the reference's feature materialisation
(`mfseg.postproc`, postproc.py:20-227).

  merge_clusters  -> mfseg_merge        union-find over eligible pairs, smallest
                                        id root; merged rows in the reference's
                                        summation order (bit-identical)
  build_features  -> mfseg_relabel + mfseg_traj_split + mfseg_voxel_csr +
                     mfseg_feature_stats
  feature_stats   -> mfseg_feature_stats (exact sums; bbox exact)

Trajectory splitting (postproc.py:152-160, 176-191) orders the points by
(traj_id, t) and finds the run breaks on the GPU; only the Python lists of
polylines / isolated points the API returns are built on the host.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field as dc_field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .engine import (DeviceField, DevicePoints, device, field_to_device, points_to_device,
                     stream_ptr, to_dev)
from .model import DELTA, ClusterCenter, FieldSet, PointSet, Segmentation


def _pct_diff(a: float, b: float) -> float:
    """Symmetric percent difference with a zero guard (postproc.py:40-42)."""
    return 2.0 * abs(a - b) / (abs(a) + abs(b) + DELTA)


def _values_match(a, b, eps_m) -> bool:
    if a is None and b is None:
        return True
    if a is None or b is None:
        return False
    return _pct_diff(a, b) <= eps_m


def merge_eligible(a: ClusterCenter, b: ClusterCenter, eps_m: float) -> bool:
    """Both averages must match within eps_m (postproc.py:53-56)."""
    return _values_match(a.p_c, b.p_c, eps_m) and _values_match(a.f_c, b.f_c, eps_m)


def merge_clusters(centers: Sequence[ClusterCenter], eps_m: float):
    """Transitive-closure merge over the pairwise value criterion (postproc.py:59-79).

    Returns (merge_map, merged centre table) exactly as the reference does.
    """
    centers = sorted(centers, key=lambda c: c.id)
    n = len(centers)
    if n == 0:
        return {}, []
    lib = N.load()
    dev = device()
    ids = to_dev(np.array([c.id for c in centers], np.int64), torch.int32, dev)
    loc = to_dev(np.array([[c.x_c, c.y_c, c.z_c, c.t_c] for c in centers], float).T.copy(), dev=dev)
    nan = float("nan")
    pc = to_dev(np.array([nan if c.p_c is None else c.p_c for c in centers], float), dev=dev)
    fc = to_dev(np.array([nan if c.f_c is None else c.f_c for c in centers], float), dev=dev)
    npt = to_dev(np.array([c.n_points for c in centers], np.int64), torch.int64, dev)
    nfl = to_dev(np.array([c.n_fields for c in centers], np.int64), torch.int64, dev)
    rep = torch.empty(n, dtype=torch.int32, device=dev)
    m_ids = torch.empty(n, dtype=torch.int32, device=dev)
    m_loc = torch.empty(4 * n, dtype=torch.float64, device=dev)
    m_p = torch.empty(n, dtype=torch.float64, device=dev)
    m_f = torch.empty(n, dtype=torch.float64, device=dev)
    m_np = torch.empty(n, dtype=torch.int64, device=dev)
    m_nf = torch.empty(n, dtype=torch.int64, device=dev)
    G = C.c_int32(0)
    ws_bytes = lib.mfseg_merge_workspace_size(n)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    N.check(lib.mfseg_merge(n, N.ptr(ids), N.ptr(loc), N.ptr(pc), N.ptr(fc), N.ptr(npt),
                            N.ptr(nfl), float(eps_m), N.ptr(rep), N.ptr(m_ids), N.ptr(m_loc),
                            N.ptr(m_p), N.ptr(m_f), N.ptr(m_np), N.ptr(m_nf), C.byref(G),
                            N.ptr(ws), ws_bytes, stream_ptr()), "mfseg_merge")
    g = G.value
    rep_h = rep.cpu().numpy()
    merge_map = {int(c.id): int(r) for c, r in zip(centers, rep_h)}
    mi, ml = m_ids[:g].cpu().numpy(), m_loc[:4 * g].cpu().numpy().reshape(4, g)
    mp, mf = m_p[:g].cpu().numpy(), m_f[:g].cpu().numpy()
    mnp, mnf = m_np[:g].cpu().numpy(), m_nf[:g].cpu().numpy()
    merged = [ClusterCenter(int(mi[j]), float(ml[0, j]), float(ml[1, j]), float(ml[2, j]),
                            float(ml[3, j]), None if np.isnan(mp[j]) else float(mp[j]),
                            None if np.isnan(mf[j]) else float(mf[j]), int(mnp[j]), int(mnf[j]))
              for j in range(g)]
    return merge_map, merged


@dataclass(frozen=True)
class FeatureStats:
    """postproc.py:95-112."""

    bbox_min: tuple
    bbox_max: tuple
    p_mean: Optional[float]
    p_std: Optional[float]
    f_mean: Optional[float]
    f_std: Optional[float]
    n_points: int
    n_fields: int

    def to_dict(self) -> dict:
        return {"bbox_min": list(self.bbox_min), "bbox_max": list(self.bbox_max),
                "p_mean": self.p_mean, "p_std": self.p_std, "f_mean": self.f_mean,
                "f_std": self.f_std, "n_points": self.n_points, "n_fields": self.n_fields}


@dataclass
class Feature:
    """One merged cluster materialised for exploration (postproc.py:115-129)."""

    id: int
    member_clusters: list
    polylines: list = dc_field(default_factory=list)
    isolated_points: list = dc_field(default_factory=list)
    voxels: dict = dc_field(default_factory=dict)
    stats: Optional[FeatureStats] = None


def _stats_from_row(row) -> FeatureStats:
    def opt(x):
        return None if np.isnan(x) else float(x)
    return FeatureStats(tuple(float(x) for x in row[0:4]), tuple(float(x) for x in row[4:8]),
                        opt(row[8]), opt(row[9]), opt(row[10]), opt(row[11]), int(row[12]),
                        int(row[13]))


def feature_slots_device(labels: torch.Tensor, lut: np.ndarray) -> torch.Tensor:
    """label -> dense feature slot on the device (mfseg_relabel)."""
    lib = N.load()
    out = torch.empty_like(labels)
    if labels.numel():
        lt = to_dev(lut.astype(np.int64), torch.int32, labels.device)
        N.check(lib.mfseg_relabel(N.ptr(labels), labels.numel(), N.ptr(lt), len(lut), N.ptr(out),
                                  stream_ptr()), "mfseg_relabel")
    return out


def feature_stats_device(n_slots: int, fld: DeviceField, fslot: Optional[torch.Tensor],
                         pts: DevicePoints, pslot: Optional[torch.Tensor]) -> np.ndarray:
    """(n_slots, 14) rows: bbox_min[4], bbox_max[4], p_mean, p_std, f_mean, f_std, n_p, n_f."""
    lib = N.load()
    dev = fld.values.device if fld.values.numel() else pts.t.device
    stats = torch.empty((n_slots, N.STAT_WORDS), dtype=torch.float64, device=dev)
    ws_bytes = lib.mfseg_feature_stats_workspace_size(n_slots)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    fs, ps = fld.struct(), pts.struct()
    N.check(lib.mfseg_feature_stats(n_slots, C.byref(fs),
                                    N.ptr(fslot) if fslot is not None and fld.nt else None,
                                    C.byref(ps),
                                    N.ptr(pslot) if pslot is not None and pts.n else None,
                                    N.ptr(stats), N.ptr(ws), ws_bytes, stream_ptr()),
            "mfseg_feature_stats")
    return stats.cpu().numpy()


def voxel_csr_device(fslot: torch.Tensor, nt: int, ncell: int, n_slots: int):
    """Per (timestep, slot) ascending cell lists: (seg_start int64 [(nt*ns)+1], cells int32)."""
    lib = N.load()
    dev = fslot.device
    seg = torch.empty(nt * n_slots + 1, dtype=torch.int64, device=dev)
    cells = torch.empty(nt * ncell, dtype=torch.int32, device=dev)
    ident = to_dev(np.arange(n_slots, dtype=np.int64), torch.int32, dev)
    ws_bytes = lib.mfseg_voxel_csr_workspace_size(nt * ncell, nt, n_slots)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    N.check(lib.mfseg_voxel_csr(N.ptr(fslot), nt, ncell, N.ptr(ident), n_slots, n_slots,
                                N.ptr(seg), N.ptr(cells), N.ptr(ws), ws_bytes, stream_ptr()),
            "mfseg_voxel_csr")
    return seg, cells


def split_trajectories_device(traj_id: torch.Tensor, t: torch.Tensor, label: torch.Tensor):
    """GPU trajectory split (postproc.py:152-160, 176-191) through mfseg_traj_split:
    returns (order, run_start, stride) with order = point indices sorted by
    (traj_id, t), run_start delimiting the runs (device tensors)."""
    lib = N.load()
    n = int(t.numel())
    dev = t.device
    order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    starts = torch.empty(n + 1, dtype=torch.int32, device=dev)
    ws = torch.empty(int(lib.mfseg_traj_split_workspace_size(n)), dtype=torch.uint8, device=dev)
    nr, stride = C.c_int64(0), C.c_double(0.0)
    tid = traj_id.to(device=dev, dtype=torch.int64).contiguous()
    lab = label.to(device=dev, dtype=torch.int32).contiguous()
    tt = t.to(device=dev, dtype=torch.float64).contiguous()
    N.check(lib.mfseg_traj_split(n, N.ptr(tid), N.ptr(tt), N.ptr(lab), N.ptr(order), N.ptr(starts),
                                 C.byref(nr), C.byref(stride), N.ptr(ws), ws.numel(), stream_ptr()),
            "mfseg_traj_split")
    return order[:n], starts[:nr.value + 1], stride.value


def _split_trajectories(fid_of_slot, pslot, traj_id, t, feats):
    """Polylines / isolated points per time-ordered trajectory (postproc.py:152-160,
    176-191): ordering and run detection on the GPU, list building on the host."""
    order, starts, _ = split_trajectories_device(traj_id, t, pslot)
    order_h = order.cpu().numpy().astype(np.int64)
    st = starts.cpu().numpy().astype(np.int64)
    if len(st) < 2:
        return
    run_fid = fid_of_slot[pslot.cpu().numpy()[order_h[st[:-1]]]]
    poly = np.diff(st) >= 2
    by_fid = np.argsort(run_fid, kind="stable")  # runs grouped by feature, order kept
    fs = run_fid[by_fid]
    bounds = np.flatnonzero(np.r_[True, fs[1:] != fs[:-1], True])
    for b0, b1 in zip(bounds[:-1].tolist(), bounds[1:].tolist()):
        f = feats[int(fs[b0])]
        sel = by_fid[b0:b1]
        ps = sel[poly[sel]]
        # polylines are views of the ordered index array (as np.split in the reference)
        f.polylines.extend(map(order_h.__getitem__, map(slice, st[ps].tolist(), st[ps + 1].tolist())))
        f.isolated_points.extend(order_h[st[sel[~poly[sel]]]].tolist())


def build_features(seg: Segmentation, merge_map: Optional[dict], points: PointSet,
                   fields: FieldSet) -> list:
    """Assemble Features: split trajectories, bucket voxels per timestep and
    compute statistics (postproc.py:136-173)."""
    if merge_map is None:
        merge_map = {c.id: c.id for c in seg.centers}
    members = {}
    for c in seg.centers:
        members.setdefault(merge_map[c.id], []).append(c.id)
    fids = sorted(members)
    feats = {f: Feature(f, sorted(members[f])) for f in fids}
    slot_of_fid = {f: s for s, f in enumerate(fids)}
    K = max([int(k) for k in merge_map] + [int(l) for l in np.asarray(seg.point_labels)[:1]] +
            [int(l) for l in np.asarray(seg.field_labels)[:1]] + [0]) + 1
    K = max(K, int(np.max(seg.point_labels, initial=0)) + 1, int(np.max(seg.field_labels, initial=0)) + 1)
    lut = np.full(K, -1, np.int64)
    for cid, rep in merge_map.items():
        if int(cid) < K:
            lut[int(cid)] = slot_of_fid.get(rep, -1)
    dev = device()
    pts = points_to_device(points, dev)
    fld = field_to_device(fields, dev)
    n_slots = len(fids)
    pslot = fslot = None
    if pts.n:
        pl = to_dev(np.asarray(seg.point_labels), torch.int32, dev)
        pslot = feature_slots_device(pl, lut)
        ps_h = pslot.cpu().numpy()
        if np.any(ps_h < 0):
            raise KeyError("point label without a merge_map entry")
        _split_trajectories(np.asarray(fids), pslot,
                            to_dev(np.asarray(points.traj_id, np.int64), torch.int64, dev), pts.t,
                            feats)
    if fld.nt:
        fl = to_dev(np.asarray(seg.field_labels), torch.int32, dev)
        fslot = feature_slots_device(fl, lut)
        ncell = int(np.prod(fld.dims))
        seg_start, cells = voxel_csr_device(fslot, fld.nt, ncell, n_slots)
        ss, ch = seg_start.cpu().numpy(), cells.cpu().numpy().astype(np.int64)
        for m in range(fld.nt):
            for s, f in enumerate(fids):
                a, b = ss[m * n_slots + s], ss[m * n_slots + s + 1]
                if b > a:
                    feats[f].voxels[m] = ch[a:b]
    rows = feature_stats_device(n_slots, fld, fslot, pts, pslot) if n_slots else []
    out = [feats[f] for f in fids]
    for s, f in enumerate(out):
        if rows[s][12] + rows[s][13] == 0:
            raise ValueError(f"feature {f.id} has no member samples")
        f.stats = _stats_from_row(rows[s])
    return out


def feature_stats(feature: Feature, points: PointSet, fields: FieldSet) -> FeatureStats:
    """Statistics of one materialised feature (postproc.py:194-227)."""
    dev = device()
    pidx = np.concatenate([np.concatenate(feature.polylines) if feature.polylines
                           else np.empty(0, np.int64),
                           np.asarray(feature.isolated_points, np.int64)]).astype(np.int64)
    pts = points_to_device(points, dev)
    fld = field_to_device(fields, dev)
    pslot = fslot = None
    if pts.n:
        ps = np.full(pts.n, -1, np.int64)
        ps[pidx] = 0
        pslot = to_dev(ps, torch.int32, dev)
    if fld.nt:
        ncell = int(np.prod(fld.dims))
        fs_h = np.full(fld.nt * ncell, -1, np.int64)
        for m, cells in feature.voxels.items():
            fs_h[int(m) * ncell + np.asarray(cells, np.int64)] = 0
        fslot = to_dev(fs_h, torch.int32, dev)
    row = feature_stats_device(1, fld, fslot, pts, pslot)[0]
    if row[12] + row[13] == 0:
        raise ValueError(f"feature {feature.id} has no member samples")
    return _stats_from_row(row)
