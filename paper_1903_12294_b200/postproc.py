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
import sys
from dataclasses import dataclass, field as dc_field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .engine import (DeviceField, DevicePoints, device, download, field_to_device,
                     points_to_device, stream_ptr, to_dev)
from .model import DELTA, ClusterCenter, FieldSet, PointSet, Segmentation


# The reference sums merged p_c / f_c with the builtin sum() (postproc.py:85-88),
# which CPython 3.12 made compensated (Neumaier); the kernel follows the running
# interpreter so merged tables stay bit-identical to the reference under it.
NEUMAIER = 1 if sys.version_info >= (3, 12) else 0


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
                            N.ptr(nfl), float(eps_m), NEUMAIER, N.ptr(rep), N.ptr(m_ids), N.ptr(m_loc),
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


def merge_device(state: dict, eps_m: float):
    """merge_clusters (postproc.py:59-92) on a device centre state (engine
    DeviceRun.state): the live rows (n_points + n_fields > 0, ascending id,
    engine.py:72-86) are compacted on the device and merged there, without the
    host table round trip.  Returns (ids, rep, merged) device tensors: ids of the
    live rows, their representative (the merge map), and the merged table
    (ids, loc [4][g], p_c, f_c, n_points, n_fields; NaN = absent)."""
    lib = N.load()
    dev = state["loc"].device
    live = torch.nonzero((state["n_points"] + state["n_fields"]) > 0).flatten()
    n = int(live.numel())
    ids = live.to(torch.int32)
    loc = state["loc"][:, live].contiguous()
    nan = torch.tensor(float("nan"), dtype=torch.float64, device=dev)
    pc = torch.where(state["has_p"][live] != 0, state["pval"][live], nan).contiguous()
    fc = torch.where(state["has_f"][live] != 0, state["fval"][live], nan).contiguous()
    npt = state["n_points"][live].contiguous()
    nfl = state["n_fields"][live].contiguous()
    rep = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    m_ids = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    m_loc = torch.empty(4 * max(n, 1), dtype=torch.float64, device=dev)
    m_p = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    m_f = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    m_np = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    m_nf = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    G = C.c_int32(0)
    if n:
        ws_bytes = lib.mfseg_merge_workspace_size(n)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        N.check(lib.mfseg_merge(n, N.ptr(ids), N.ptr(loc), N.ptr(pc), N.ptr(fc), N.ptr(npt),
                                N.ptr(nfl), float(eps_m), NEUMAIER, N.ptr(rep), N.ptr(m_ids), N.ptr(m_loc),
                                N.ptr(m_p), N.ptr(m_f), N.ptr(m_np), N.ptr(m_nf), C.byref(G),
                                N.ptr(ws), ws_bytes, stream_ptr()), "mfseg_merge")
    g = G.value
    merged = {"ids": m_ids[:g], "loc": m_loc[:4 * g].reshape(4, g), "p_c": m_p[:g], "f_c": m_f[:g],
              "n_points": m_np[:g], "n_fields": m_nf[:g]}
    return ids, rep[:n], merged


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
    """Per (timestep, slot) ascending cell lists: (seg_start int64 [(nt*ns)+1], cells int32).
    Timesteps are processed in groups of < 2^31 samples (one call each)."""
    lib = N.load()
    dev = fslot.device
    seg = torch.empty(nt * n_slots + 1, dtype=torch.int64, device=dev)
    cells = torch.empty(nt * ncell, dtype=torch.int32, device=dev)
    ident = to_dev(np.arange(n_slots, dtype=np.int64), torch.int32, dev)
    per = max(1, min(nt, ((1 << 31) - 1) // max(ncell, 1)))
    ws_bytes = lib.mfseg_voxel_csr_workspace_size(per * ncell, per, n_slots)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    part = torch.empty(per * n_slots + 1, dtype=torch.int64, device=dev) if per < nt else seg
    for m0 in range(0, nt, per):
        m1 = min(nt, m0 + per)
        dst = seg if per >= nt else part
        N.check(lib.mfseg_voxel_csr(N.ptr(fslot[m0 * ncell:]), m1 - m0, ncell, N.ptr(ident),
                                    n_slots, n_slots, N.ptr(dst), N.ptr(cells[m0 * ncell:]),
                                    N.ptr(ws), ws_bytes, stream_ptr()), "mfseg_voxel_csr")
        if per < nt:   # offsets of this group are relative to its first sample
            seg[m0 * n_slots:m1 * n_slots] = part[:(m1 - m0) * n_slots] + m0 * ncell
    if per < nt:
        seg[nt * n_slots] = nt * ncell
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
    if starts.numel() < 2:
        return
    order_h = download(order, torch.int64)
    st = download(starts, torch.int64)
    run_fid = fid_of_slot[download(pslot[order[starts[:-1].long()].long()])]
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


def _feature_slots(seg: Segmentation, merge_map: Optional[dict]):
    """(feature ids ascending, Feature per id, label -> slot lut) (postproc.py:141-150)."""
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
    return fids, feats, lut


def build_features(seg: Segmentation, merge_map: Optional[dict], points: PointSet,
                   fields: FieldSet) -> list:
    """Assemble Features: split trajectories, bucket voxels per timestep and
    compute statistics (postproc.py:136-173)."""
    fids, feats, lut = _feature_slots(seg, merge_map)
    dev = device()
    pts = points_to_device(points, dev)
    fld = field_to_device(fields, dev)
    n_slots = len(fids)
    pslot = fslot = None
    if pts.n:
        pl = to_dev(np.asarray(seg.point_labels), torch.int32, dev)
        pslot = feature_slots_device(pl, lut)
        if bool((pslot < 0).any()):
            raise KeyError("point label without a merge_map entry")
        _split_trajectories(np.asarray(fids), pslot,
                            to_dev(np.asarray(points.traj_id, np.int64), torch.int64, dev), pts.t,
                            feats)
    if fld.nt:
        fl = to_dev(np.asarray(seg.field_labels), torch.int32, dev)
        fslot = feature_slots_device(fl, lut)
        ncell = int(np.prod(fld.dims))
        seg_start, cells = voxel_csr_device(fslot, fld.nt, ncell, n_slots)
        ss, ch = seg_start.cpu().numpy(), download(cells, torch.int64)
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


# ============================================================== sharded feature materialisation
#
# build_features over samples sharded across ranks (parallel.py): each rank
# holds a slab of the field and the point samples of its bins.  Statistics are
# exact integer partials reduced across ranks (bit-identical for any rank
# count); voxel lists stay with the rank that owns the cells (keyed by global
# timestep, cells as global flat indices); trajectories are shuffled to an
# owner rank by contiguous trajectory-id ranges (one all-to-all) and split
# there with the common stride of all point times, so every polyline is whole.
# The union over ranks, concatenated in rank order, equals build_features on
# the whole dataset, in the reference's order.

M42 = (1 << 42) - 1


def fix128_to_limbs(words: torch.Tensor) -> torch.Tensor:
    """(n, 2) int64 (lo, hi) pairs of 128-bit two's complement values -> (n, 3)
    limbs of 42 / 42 / 44 bits whose sums over < 2^20 ranks are exact."""
    lo, hi = words[:, 0], words[:, 1]
    l0 = lo & M42
    l1 = ((lo >> 42) & ((1 << 22) - 1)) | ((hi & ((1 << 20) - 1)) << 22)
    l2 = hi >> 20
    return torch.stack([l0, l1, l2], dim=1)


def limbs_to_fix128(limbs: torch.Tensor) -> torch.Tensor:
    """Inverse of fix128_to_limbs after a SUM (carries propagated)."""
    l0, l1, l2 = limbs[:, 0].clone(), limbs[:, 1].clone(), limbs[:, 2].clone()
    c = l0 >> 42
    l0 = l0 & M42
    l1 = l1 + c
    c = l1 >> 42
    l1 = l1 & M42
    l2 = l2 + c
    lo = l0 | (l1 << 42)
    hi = (l1 >> 22) | (l2 << 20)
    return torch.stack([lo, hi], dim=1)


_SIGN = -(1 << 63)


def reduce_stat_partials(S: torch.Tensor, group=None) -> None:
    """In-place cross-rank reduction of mfseg_feature_stats_pass partials
    ([n][18] int64 views of the uint64 words): 128-bit sums (words 0..7) as
    exact limb sums, counts (8, 9) summed, bbox keys (10..13 min, 14..17 max)
    reduced in unsigned order."""
    import torch.distributed as dist
    n = S.shape[0]
    if n == 0:
        return
    pairs = S[:, 0:8].reshape(-1, 2)
    limbs = fix128_to_limbs(pairs)
    dist.all_reduce(limbs, op=dist.ReduceOp.SUM, group=group)
    S[:, 0:8] = limbs_to_fix128(limbs).reshape(n, 8)
    cnt = S[:, 8:10].contiguous()
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
    S[:, 8:10] = cnt
    for a, b, op in ((10, 14, dist.ReduceOp.MIN), (14, 18, dist.ReduceOp.MAX)):
        keys = S[:, a:b] ^ _SIGN            # unsigned order -> signed order
        keys = keys.contiguous()
        dist.all_reduce(keys, op=op, group=group)
        S[:, a:b] = keys ^ _SIGN


def feature_stats_sharded(n_slots: int, fld: DeviceField, fslot, pts: DevicePoints, pslot,
                          group=None) -> np.ndarray:
    """feature_stats rows over all ranks' samples (postproc.py:194-227): two
    staged passes with exact partials reduced between them."""
    lib = N.load()
    dev = fld.values.device if fld.values.numel() else pts.t.device
    S = torch.empty((n_slots, N.STAT_PARTIAL_WORDS), dtype=torch.int64, device=dev)
    mean = torch.empty((n_slots, 2), dtype=torch.float64, device=dev)
    stats = torch.empty((n_slots, N.STAT_WORDS), dtype=torch.float64, device=dev)
    fs, ps = fld.struct(), pts.struct()
    fp = N.ptr(fslot) if fslot is not None and fld.nt else None
    pp = N.ptr(pslot) if pslot is not None and pts.n else None
    backend_cpu = _exchange_on_cpu(group)

    def reduce_(t):
        if backend_cpu:
            h = t.cpu()
            reduce_stat_partials(h, group)
            t.copy_(h)
        else:
            reduce_stat_partials(t, group)

    N.check(lib.mfseg_feature_stats_pass(n_slots, C.byref(fs), fp, C.byref(ps), pp, 0, None,
                                         N.ptr(S), stream_ptr()), "mfseg_feature_stats_pass")
    reduce_(S)
    N.check(lib.mfseg_feature_stats_means(n_slots, N.ptr(S), N.ptr(mean), stream_ptr()),
            "mfseg_feature_stats_means")
    S1 = torch.zeros_like(S)          # pass 1 adds the squared deviations into words 4..7
    S1[:, 10:14] = -1                 # (keep the bbox words neutral for the reduction)
    N.check(lib.mfseg_feature_stats_pass(n_slots, C.byref(fs), fp, C.byref(ps), pp, 1,
                                         N.ptr(mean), N.ptr(S1), stream_ptr()),
            "mfseg_feature_stats_pass")
    reduce_(S1)
    S[:, 4:8] = S1[:, 4:8]
    N.check(lib.mfseg_feature_stats_final(n_slots, N.ptr(S), N.ptr(mean), N.ptr(stats),
                                          stream_ptr()), "mfseg_feature_stats_final")
    return stats.cpu().numpy()


def _exchange_on_cpu(group) -> bool:
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def global_stride(t: torch.Tensor, group=None) -> float:
    """min positive difference of the unique point times of all ranks
    (postproc.py:152-154); +inf with fewer than two unique times."""
    import torch.distributed as dist
    u = torch.unique(t).cpu().numpy() if t.numel() else np.zeros(0)
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, u, group=group)
    allu = np.unique(np.concatenate(parts)) if parts else np.zeros(0)
    return float(np.diff(allu).min()) if len(allu) > 1 else float("inf")


def traj_owner_bounds(tmin: int, tmax: int, world: int) -> np.ndarray:
    """Owner ranges of trajectory ids: rank r owns [b[r], b[r + 1]), contiguous
    and increasing with the rank (so rank-order concatenation keeps the
    reference's (traj_id, t) run order)."""
    span = tmax - tmin + 1
    return np.array([tmin + (span * r) // world for r in range(world + 1)], dtype=np.int64)


def exchange_by_trajectory(traj_id: torch.Tensor, cols, group=None):
    """All-to-all of the point samples to the rank owning their trajectory.
    `cols`: list of 1-D tensors aligned with traj_id.  Returns (traj_id, cols)
    of the samples this rank owns, ordered by source rank then source order."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    cpu = _exchange_on_cpu(group)
    dev = torch.device("cpu") if cpu else traj_id.device
    tid = traj_id.to(dev)
    cols = [c.to(dev) for c in cols]
    lo = int(tid.min()) if tid.numel() else np.iinfo(np.int64).max
    hi = int(tid.max()) if tid.numel() else np.iinfo(np.int64).min
    mm = torch.tensor([lo, -hi], dtype=torch.int64, device=dev)
    dist.all_reduce(mm, op=dist.ReduceOp.MIN, group=group)
    if int(mm[0]) > -int(mm[1]):       # no points anywhere
        return tid, cols
    bounds = torch.as_tensor(traj_owner_bounds(int(mm[0]), -int(mm[1]), world), device=dev)
    owner = torch.bucketize(tid, bounds[1:-1], right=True)
    order = torch.argsort(owner, stable=True)
    send = torch.bincount(owner, minlength=world).to(torch.int64)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    s_sizes, r_sizes = send.tolist(), recv.tolist()
    out = []
    for c in [tid] + cols:
        src = c[order].contiguous()
        dst = torch.empty(sum(r_sizes), dtype=c.dtype, device=dev)
        dist.all_to_all_single(dst, src, r_sizes, s_sizes, group=group)
        out.append(dst)
    return out[0], out[1:]


def build_features_sharded(seg: Segmentation, merge_map: Optional[dict], points, fields,
                           group=None, point_index=None, field_offset=(0, 0, 0),
                           timestep_offset: int = 0, grid_dims=None) -> list:
    """build_features (postproc.py:136-173) over sharded samples: `seg` holds
    this rank's labels (and the replicated centre table), `points` / `fields`
    this rank's samples (see parallel.shard_dataset); `point_index` the global
    indices of the local points (default: local order), `field_offset` /
    `grid_dims` the slab's first cell and the whole grid (spatial slabs),
    `timestep_offset` the global index of the first local timestep (time slabs).

    Every rank returns all features with global statistics; voxels of its own
    cells (global timestep keys, global flat cell indices) and the polylines /
    isolated points of the trajectories it owns (global point indices)."""
    fids, feats, lut = _feature_slots(seg, merge_map)
    dev = device()
    pts = points_to_device(points, dev)
    fld = field_to_device(fields, dev)
    fld.offset = tuple(int(o) for o in field_offset)
    n_slots = len(fids)
    pslot = fslot = None
    if pts.n:
        pl = to_dev(np.asarray(seg.point_labels), torch.int32, dev)
        pslot = feature_slots_device(pl, lut)
        if bool((pslot < 0).any()):
            raise KeyError("point label without a merge_map entry")
    gidx = torch.as_tensor(np.arange(pts.n) if point_index is None else np.asarray(point_index),
                           dtype=torch.int64, device=dev)
    # trajectories: shuffle to owners, split there with the common stride
    stride = global_stride(pts.t, group)
    tid = to_dev(np.asarray(points.traj_id, np.int64) if pts.n else np.zeros(0, np.int64),
                 torch.int64, dev)
    o_tid, (o_t, o_slot, o_gidx) = exchange_by_trajectory(
        tid, [pts.t, pslot if pslot is not None else torch.zeros(0, dtype=torch.int32, device=dev),
              gidx], group)
    if o_tid.numel():
        _split_owned(np.asarray(fids), o_tid.to(dev), o_t.to(dev), o_slot.to(dev), o_gidx.to(dev),
                     stride, feats)
    # voxels of the local cells
    if fld.nt:
        fl = to_dev(np.asarray(seg.field_labels), torch.int32, dev)
        fslot = feature_slots_device(fl, lut)
        nx, ny, nz = fld.dims
        ncell = nx * ny * nz
        gd = tuple(grid_dims) if grid_dims is not None else (nx, ny, nz)
        seg_start, cells = voxel_csr_device(fslot, fld.nt, ncell, n_slots)
        ss, ch = seg_start.cpu().numpy(), cells.cpu().numpy().astype(np.int64)
        x0, y0, z0 = fld.offset
        if (x0, y0, z0) != (0, 0, 0) or gd != (nx, ny, nz):
            i, r = ch % nx, ch // nx
            j, k = r % ny, r // ny
            ch = (i + x0) + gd[0] * ((j + y0) + gd[1] * (k + z0))
        for m in range(fld.nt):
            for s_, f in enumerate(fids):
                a, b = ss[m * n_slots + s_], ss[m * n_slots + s_ + 1]
                if b > a:
                    feats[f].voxels[m + timestep_offset] = ch[a:b]
    rows = feature_stats_sharded(n_slots, fld, fslot, pts, pslot, group) if n_slots else []
    out = [feats[f] for f in fids]
    for s_, f in enumerate(out):
        if rows[s_][12] + rows[s_][13] == 0:
            raise ValueError(f"feature {f.id} has no member samples")
        f.stats = _stats_from_row(rows[s_])
    return out


def _split_owned(fid_of_slot, tid, t, slot, gidx, stride, feats):
    """The owner's split of whole trajectories (postproc.py:152-160, 176-191)
    with the common stride; polylines hold global point indices."""
    lib = N.load()
    n = int(t.numel())
    dev = t.device
    order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    starts = torch.empty(n + 1, dtype=torch.int32, device=dev)
    ws = torch.empty(int(lib.mfseg_traj_split_workspace_size(n)), dtype=torch.uint8, device=dev)
    nr = C.c_int64(0)
    tid = tid.to(torch.int64).contiguous()
    slot = slot.to(torch.int32).contiguous()
    t = t.to(torch.float64).contiguous()
    N.check(lib.mfseg_traj_split_stride(n, N.ptr(tid), N.ptr(t), N.ptr(slot), float(stride),
                                        N.ptr(order), N.ptr(starts), C.byref(nr), N.ptr(ws),
                                        ws.numel(), stream_ptr()), "mfseg_traj_split_stride")
    order_h = order[:n].cpu().numpy().astype(np.int64)
    st = starts[:nr.value + 1].cpu().numpy().astype(np.int64)
    g = gidx.cpu().numpy()[order_h]            # global indices in (traj, t) order
    if len(st) < 2:
        return
    run_fid = fid_of_slot[slot.cpu().numpy()[order_h[st[:-1]]]]
    poly = np.diff(st) >= 2
    by_fid = np.argsort(run_fid, kind="stable")
    fs = run_fid[by_fid]
    bounds = np.flatnonzero(np.r_[True, fs[1:] != fs[:-1], True])
    for b0, b1 in zip(bounds[:-1].tolist(), bounds[1:].tolist()):
        f = feats[int(fs[b0])]
        sel = by_fid[b0:b1]
        ps = sel[poly[sel]]
        f.polylines.extend(map(g.__getitem__, map(slice, st[ps].tolist(), st[ps + 1].tolist())))
        f.isolated_points.extend(g[st[sel[~poly[sel]]]].tolist())
