"""CPU ORACLE for the segmentation hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm (arXiv 1903.12294,
reference package `mfseg` under /root/reference/pkg/src).  It exists to CHECK the
CUDA product path and to provide the CPU baseline arm of `bench.py`.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py` (cpu_baseline / --impl
reference) may import it.  The product package `paper_1903_12294_b200` never
imports, links or calls anything under `oracle/`.

Parity pinning: every function here is checked against golden vectors produced
by running the reference itself (tests/golden/make_golden.py → tests/golden/*.npz,
and the recorded frontend fixtures), see tests/test_oracle_golden.py.

Arithmetic contract (identical to the reference, op for op):
  * cell centre      x = origin + (i + 0.5) * spacing          model.py:137-142
  * seed             x = min + (j + 0.5) * C                   engine.py:31-45
  * bin              clip(floor((x - min) / C), 0, k-1)        engine.py:111-117
  * metric           d = c - s; sst = sqrt(((d0²+d1²)+d2²)+(cf·d3)²);
                     D = wv·|v - c_v|·[has] + wd·sst           engine.py:137-149
  * window           3^4 neighbour bins ∧ |c - s| ≤ C per axis engine.py:119-131,179-181
  * argmin           first minimum over ascending ids           engine.py:184
  * fallback         doubling box over all K centres           engine.py:195-205
  * accumulate       np.bincount (sequential, index order)      engine.py:244-263
"""

from __future__ import annotations

import itertools
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field as dc_field
from typing import Callable, Optional

import numpy as np

DELTA = 1e-12   # model.py:16


# ============================================================== geometry

def interval_lengths(mins: np.ndarray, maxs: np.ndarray, k) -> np.ndarray:
    """C_d = (max_d - min_d) / k_d                           (model.py:275-280)."""
    return (np.asarray(maxs, float) - np.asarray(mins, float)) / np.asarray(k)


def seed_locations(mins: np.ndarray, C: np.ndarray, k) -> np.ndarray:
    """(K,4) seeds, ids t-major then z, y, x (x fastest)     (engine.py:31-45)."""
    kx, ky, kz, kt = (int(v) for v in k)
    ax = [mins[d] + (np.arange(int(k[d])) + 0.5) * C[d] for d in range(4)]
    it, iz, iy, ix = np.meshgrid(np.arange(kt), np.arange(kz), np.arange(ky), np.arange(kx),
                                 indexing="ij")
    return np.column_stack([ax[0][ix.ravel()], ax[1][iy.ravel()], ax[2][iz.ravel()],
                            ax[3][it.ravel()]])


def cell_centres(dims, origin, spacing) -> np.ndarray:
    """(n_cells,3) centres, flat index i + nx*(j + ny*k)      (model.py:137-142)."""
    nx, ny, nz = (int(v) for v in dims)
    flat = np.arange(nx * ny * nz)
    ijk = np.column_stack([flat % nx, (flat // nx) % ny, flat // (nx * ny)])
    return np.asarray(origin, float) + (ijk + 0.5) * np.asarray(spacing, float)


def field_locations(dims, origin, spacing, times) -> np.ndarray:
    """(T*n_cells,4) sample locations, timestep-major       (model.py:144-150)."""
    cc = cell_centres(dims, origin, spacing)
    times = np.asarray(times, float)
    if len(times) == 0:
        return np.empty((0, 4))
    return np.column_stack([np.tile(cc, (len(times), 1)), np.repeat(times, len(cc))])


def bins_of(loc: np.ndarray, mins, C, k) -> np.ndarray:
    """clip(floor((loc - min)/C), 0, k-1) per axis            (engine.py:111-113)."""
    b = np.floor((loc - mins) / C).astype(np.int64)
    return np.clip(b, 0, np.asarray(k) - 1)


def flatten_bins(b: np.ndarray, k) -> np.ndarray:
    kx, ky, kz, _ = (int(v) for v in k)
    return ((b[..., 3] * kz + b[..., 2]) * ky + b[..., 1]) * kx + b[..., 0]


# ============================================================== centre state

@dataclass
class Centres:
    """Per-id centre arrays, mirror of engine.CenterState (engine.py:48-70)."""

    loc: np.ndarray
    pval: np.ndarray
    fval: np.ndarray
    has_p: np.ndarray
    has_f: np.ndarray
    n_points: np.ndarray
    n_fields: np.ndarray
    dormant: np.ndarray

    @classmethod
    def seeded(cls, seeds: np.ndarray) -> "Centres":
        K = len(seeds)
        return cls(seeds.copy(), np.full(K, np.nan), np.full(K, np.nan), np.zeros(K, bool),
                   np.zeros(K, bool), np.zeros(K, np.int64), np.zeros(K, np.int64),
                   np.zeros(K, bool))

    def live_ids(self) -> np.ndarray:
        return np.flatnonzero(self.n_points + self.n_fields > 0)


class NeighbourTable:
    """Centres bucketed by bin; candidate lists over the 3^4 neighbourhood.

    Restates engine.CenterGrid (engine.py:89-134): a centre sits in exactly one
    (clipped) bin; the candidates of a sample bin are the ascending ids of all
    centres in the in-range neighbour bins.
    """

    _OFF = np.array(list(itertools.product((-1, 0, 1), repeat=4)))

    def __init__(self, cloc, mins, C, k):
        self.mins, self.C, self.k = np.asarray(mins, float), np.asarray(C, float), np.asarray(k)
        key = flatten_bins(bins_of(cloc, self.mins, self.C, self.k), self.k)
        order = np.argsort(key, kind="stable")
        sk = key[order]
        cut = np.flatnonzero(np.r_[True, sk[1:] != sk[:-1]])
        self.members = {int(sk[a]): np.sort(order[a:b])
                        for a, b in zip(cut, np.r_[cut[1:], len(sk)])}
        self._cache = {}

    def candidates(self, b4: np.ndarray) -> np.ndarray:
        key = int(flatten_bins(b4, self.k))
        hit = self._cache.get(key)
        if hit is not None:
            return hit
        nb = b4 + self._OFF
        nb = nb[np.all((nb >= 0) & (nb < self.k), axis=1)]
        lists = [self.members.get(int(q)) for q in flatten_bins(nb, self.k)]
        lists = [x for x in lists if x is not None]
        out = np.sort(np.concatenate(lists)) if lists else np.empty(0, np.int64)
        self._cache[key] = out
        return out


# ============================================================== assignment

def distance_matrix(sloc, sval, cloc, cval, chas, wv, wd, cf) -> np.ndarray:
    """(n_samples, n_centres) D, reference op order            (engine.py:137-149)."""
    d = cloc[None, :, :] - sloc[:, None, :]
    q = d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1] + d[..., 2] * d[..., 2]
    dt = cf * d[..., 3]
    sst = np.sqrt(q + dt * dt)
    if wv > 0:
        cv = np.where(chas, cval, 0.0)
        vt = wv * np.where(chas[None, :], np.abs(sval[:, None] - cv[None, :]), 0.0)
    else:
        vt = 0.0
    return vt + wd * sst


def widen_search(sloc, sval, cloc, cval, chas, wv, wd, cf, C) -> int:
    """Stranded sample: doubling window over ALL centres       (engine.py:195-205)."""
    mult = 2.0
    while True:
        ok = np.flatnonzero(np.all(np.abs(cloc - sloc) <= mult * C, axis=1))
        if len(ok):
            D = distance_matrix(sloc[None, :], np.atleast_1d(sval), cloc[ok], cval[ok],
                                chas[ok], wv, wd, cf)[0]
            return int(ok[np.argmin(D)])
        mult *= 2.0


def _assign_block(sloc, sval, cloc, cval, chas, table: NeighbourTable, wv, wd, cf, C):
    """Windowed argmin for one block of samples            (engine.py:164-192)."""
    n = len(sloc)
    out = np.full(n, -1, np.int64)
    b = bins_of(sloc, table.mins, table.C, table.k)
    key = flatten_bins(b, table.k)
    order = np.argsort(key, kind="stable")
    sk = key[order]
    cut = np.flatnonzero(np.r_[True, sk[1:] != sk[:-1]]) if n else np.zeros(0, np.int64)
    lost = []
    for a, e in zip(cut, np.r_[cut[1:], n]):
        g = order[a:e]
        cand = table.candidates(b[g[0]])
        if len(cand) == 0:
            lost.append(g)
            continue
        inside = np.all(np.abs(cloc[cand][None, :, :] - sloc[g][:, None, :]) <= C, axis=2)
        D = distance_matrix(sloc[g], sval[g], cloc[cand], cval[cand], chas[cand], wv, wd, cf)
        D[~inside] = np.inf
        hit = inside.any(axis=1)
        out[g[hit]] = cand[np.argmin(D[hit], axis=1)]
        if not hit.all():
            lost.append(g[~hit])
    for g in lost:
        for s in g:
            out[s] = widen_search(sloc[s], sval[s], cloc, cval, chas, wv, wd, cf, C)
    return out


def assign_kind(sloc, sval, cloc, cval, chas, table, wv, wd, cf, C, workers=1, chunk=None):
    """All samples of one kind; chunks on a thread pool       (engine.py:221-241)."""
    n = len(sloc)
    out = np.empty(n, np.int64)
    if n == 0:
        return out
    step = n if not chunk else int(chunk)
    spans = [(s, min(s + step, n)) for s in range(0, n, step)]

    def one(span):
        s, e = span
        return _assign_block(sloc[s:e], sval[s:e], cloc, cval, chas, table, wv, wd, cf, C)

    if workers > 1 and len(spans) > 1:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            parts = list(pool.map(one, spans))
    else:
        parts = [one(s) for s in spans]
    for (s, e), p in zip(spans, parts):
        out[s:e] = p
    return out


# ============================================================== accumulate / update

def cluster_sums(plabels, ploc, pval, flabels, floc, fval, K):
    """Per-cluster sums with np.bincount's sequential order   (engine.py:244-263)."""
    sums = np.zeros((K, 4))
    psum, fsum = np.zeros(K), np.zeros(K)
    n_p, n_f = np.zeros(K, np.int64), np.zeros(K, np.int64)
    if len(plabels):
        for d in range(4):
            sums[:, d] += np.bincount(plabels, weights=ploc[:, d], minlength=K)
        psum += np.bincount(plabels, weights=pval, minlength=K)
        n_p += np.bincount(plabels, minlength=K)
    if len(flabels):
        for d in range(4):
            sums[:, d] += np.bincount(flabels, weights=floc[:, d], minlength=K)
        fsum += np.bincount(flabels, weights=fval, minlength=K)
        n_f += np.bincount(flabels, minlength=K)
    return sums, psum, fsum, n_p, n_f


def refresh_centres(old: Centres, sums, psum, fsum, n_p, n_f) -> Centres:
    """Member means; empty clusters keep their state, go dormant (engine.py:266-286)."""
    tot = n_p + n_f
    live = tot > 0
    loc = old.loc.copy()
    loc[live] = sums[live] / tot[live, None]
    has_p, has_f = n_p > 0, n_f > 0
    pv = np.where(has_p, psum / np.maximum(n_p, 1), np.nan)
    fv = np.where(has_f, fsum / np.maximum(n_f, 1), np.nan)
    dead = ~live
    pv[dead], fv[dead] = old.pval[dead], old.fval[dead]
    has_p[dead], has_f[dead] = old.has_p[dead], old.has_f[dead]
    return Centres(loc, pv, fv, has_p, has_f, n_p.copy(), n_f.copy(), dead)


def _rel(old, new):
    return np.abs(new - old) / (np.abs(old) + DELTA)


def is_converged(old: Centres, new: Centres, eps_c: float) -> bool:
    """Relative change < eps_c for every active centre value   (engine.py:293-307)."""
    act = ~new.dormant
    if not act.any():
        return True
    if np.any(_rel(old.loc[act], new.loc[act]) >= eps_c):
        return False
    for ov, oh, nv, nh in ((old.pval, old.has_p, new.pval, new.has_p),
                           (old.fval, old.has_f, new.fval, new.has_f)):
        if np.any(oh[act] != nh[act]):
            return False
        both = act & oh & nh
        if np.any(_rel(ov[both], nv[both]) >= eps_c):
            return False
    return True


def largest_change(old: Centres, new: Centres) -> float:
    """Progress delta                                          (engine.py:310-320)."""
    act = ~new.dormant
    if not act.any():
        return 0.0
    out = [_rel(old.loc[act], new.loc[act]).max()]
    for ov, oh, nv, nh in ((old.pval, old.has_p, new.pval, new.has_p),
                           (old.fval, old.has_f, new.fval, new.has_f)):
        both = act & oh & nh
        if both.any():
            out.append(_rel(ov[both], nv[both]).max())
    return float(max(out))


# ============================================================== full run

@dataclass
class Result:
    point_labels: np.ndarray
    field_labels: np.ndarray
    centres: Centres
    iterations_used: int
    converged: bool
    progress: list = dc_field(default_factory=list)


def segment(p_loc, p_val, f_dims, f_origin, f_spacing, f_times, f_values, mins, maxs, k,
            c_f=1.0, w_d=1.0, w_p=1.0, w_f=1.0, eps_c=0.01, max_iterations=50,
            workers=1, chunk=None, progress: Optional[Callable] = None,
            passes_cb: Optional[Callable] = None) -> Result:
    """engine.run restated (engine.py:323-381). Inputs are already normalized."""
    p_loc = np.asarray(p_loc, float).reshape(-1, 4)
    p_val = np.asarray(p_val, float)
    f_values = np.asarray(f_values, float)
    if len(p_loc) == 0 and f_values.size == 0:
        raise ValueError("no samples of either kind")
    mins, maxs = np.asarray(mins, float), np.asarray(maxs, float)
    C = interval_lengths(mins, maxs, k)
    floc = field_locations(f_dims, f_origin, f_spacing, f_times) if f_values.size else np.empty((0, 4))
    fval = f_values.reshape(-1)
    cs = Centres.seeded(seed_locations(mins, C, k))
    K = len(cs.loc)

    def one_pass(c, wd, wp, wf):
        tab = NeighbourTable(c.loc, mins, C, k)
        pl = assign_kind(p_loc, p_val, c.loc, c.pval, c.has_p, tab, wp, wd, c_f, C, workers, chunk)
        fl = assign_kind(floc, fval, c.loc, c.fval, c.has_f, tab, wf, wd, c_f, C, workers, chunk)
        if passes_cb is not None:
            passes_cb()
        return pl, fl, refresh_centres(c, *cluster_sums(pl, p_loc, p_val, fl, floc, fval, K))

    pl, fl, cs = one_pass(cs, 1.0, 0.0, 0.0)          # initial pass, engine.py:346-353
    it_used, conv, prog = 0, False, []
    for it in range(1, int(max_iterations) + 1):
        pl, fl, new = one_pass(cs, w_d, w_p, w_f)
        delta = largest_change(cs, new)
        conv = is_converged(cs, new, eps_c)
        cs, it_used = new, it
        prog.append((it, delta))
        if progress is not None:
            progress(it, delta)
        if conv:
            break
    return Result(pl.astype(np.int32), fl.astype(np.int32), cs, it_used, conv, prog)


# ============================================================== ingest

def minmax_normalize(values: np.ndarray):
    """(v - lo)/(hi - lo); a degenerate range maps to 0      (ingest.py:312-318)."""
    lo, hi = float(values.min()), float(values.max())
    if hi == lo:
        return np.zeros_like(values), lo, hi
    return (values - lo) / (hi - lo), lo, hi


def tight_extent(p_loc, f_dims, f_origin, f_spacing, f_times, pad=1e-9):
    """Bounding 4D box with padding of degenerate axes       (ingest.py:204-227)."""
    los, his = [], []
    if f_times is not None and len(f_times) > 0:
        los.append(np.concatenate([f_origin, [f_times[0]]]))
        his.append(np.concatenate([np.asarray(f_origin) + np.array(f_dims) * np.asarray(f_spacing),
                                   [f_times[-1]]]))
    if p_loc is not None and len(p_loc) > 0:
        los.append(p_loc.min(axis=0))
        his.append(p_loc.max(axis=0))
    lo, hi = np.min(los, axis=0), np.max(his, axis=0)
    span = hi - lo
    hi = np.where(span <= 0, hi + np.maximum(pad, np.abs(hi) * pad) + pad, hi)
    return lo, hi


def link_index(f_dims, f_origin, f_spacing, f_times, xyz, t):
    """(cell, interval) buckets, stable by point index      (ingest.py:261-280).

    Returns (keys (B,4) int64 sorted, sizes, members) in CSR form.
    """
    if len(t) == 0:
        return np.zeros((0, 4), np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64)
    cell = np.floor((xyz - f_origin) / f_spacing).astype(np.int64)
    if np.any(cell < 0) or np.any(cell >= np.array(f_dims)):
        raise ValueError("point sample outside the field grid")
    nint = max(len(f_times) - 1, 1)
    m = np.clip(np.searchsorted(f_times, t, side="right") - 1, 0, nint - 1)
    nx, ny, nz = (int(v) for v in f_dims)
    key = ((cell[:, 2] * ny + cell[:, 1]) * nx + cell[:, 0]) * nint + m
    order = np.argsort(key, kind="stable")
    sk = key[order]
    cut = np.flatnonzero(np.r_[True, sk[1:] != sk[:-1]])
    uk = sk[cut]
    k3, mm = uk // nint, uk % nint
    keys = np.column_stack([k3 % nx, (k3 // nx) % ny, k3 // (nx * ny), mm])
    sizes = np.diff(np.r_[cut, len(sk)])
    return keys, sizes, order


# ============================================================== post-processing

@dataclass
class Summary:
    """Centre-table row (model.py:160-190)."""

    id: int
    loc: np.ndarray
    p_c: Optional[float]
    f_c: Optional[float]
    n_points: int
    n_fields: int


def table_of(cs: Centres) -> list:
    """Live centres in id order (engine.py:72-86)."""
    return [Summary(int(i), cs.loc[i].copy(), float(cs.pval[i]) if cs.has_p[i] else None,
                    float(cs.fval[i]) if cs.has_f[i] else None, int(cs.n_points[i]),
                    int(cs.n_fields[i])) for i in cs.live_ids()]


def _pct(a, b):
    return 2.0 * abs(a - b) / (abs(a) + abs(b) + DELTA)     # postproc.py:40-42


def _match(a, b, eps):
    if a is None and b is None:
        return True
    if a is None or b is None:
        return False
    return _pct(a, b) <= eps                                 # postproc.py:45-50


def neumaier_sum(xs) -> float:
    """CPython >= 3.12 builtin sum() over floats (compensated, Neumaier).

    The reference's merged p_c / f_c are `sum(generator of floats) / n`
    (postproc.py:87-90); on the interpreter of this image (3.12.3) that sum is
    compensated, so the restatement spells the same recurrence out.
    """
    f, c = 0.0, 0.0
    for x in xs:
        t = f + x
        if abs(f) >= abs(x):
            c += (f - t) + x
        else:
            c += (x - t) + f
        f = t
    if c and np.isfinite(c):
        f += c
    return f


def merge(rows: list, eps_m: float):
    """Transitive closure over value-eligible pairs, min-id representative,
    count-weighted merged rows summed in ascending member order (postproc.py:59-92)."""
    ids = [r.id for r in rows]
    parent = {i: i for i in ids}

    def root(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for x in range(len(rows)):
        for y in range(x + 1, len(rows)):
            a, b = rows[x], rows[y]
            if _match(a.p_c, b.p_c, eps_m) and _match(a.f_c, b.f_c, eps_m):
                ra, rb = root(a.id), root(b.id)
                if ra != rb:
                    lo, hi = min(ra, rb), max(ra, rb)
                    parent[hi] = lo
    mmap = {i: root(i) for i in ids}
    groups = {}
    for r in rows:
        groups.setdefault(mmap[r.id], []).append(r)
    merged = []
    for rep in sorted(groups):
        mem = groups[rep]
        n_p = sum(r.n_points for r in mem)
        n_f = sum(r.n_fields for r in mem)
        acc = 0
        for r in mem:
            acc = acc + r.loc * (r.n_points + r.n_fields)
        loc = acc / (n_p + n_f)
        pc = fc = None
        if n_p > 0:
            pc = neumaier_sum([r.p_c * r.n_points for r in mem if r.p_c is not None]) / n_p
        if n_f > 0:
            fc = neumaier_sum([r.f_c * r.n_fields for r in mem if r.f_c is not None]) / n_f
        merged.append(Summary(rep, loc, pc, fc, n_p, n_f))
    return mmap, merged


@dataclass
class FeatureOut:
    id: int
    member_clusters: list
    polylines: list = dc_field(default_factory=list)
    isolated_points: list = dc_field(default_factory=list)
    voxels: dict = dc_field(default_factory=dict)
    stats: Optional[dict] = None


def features(rows, mmap, point_labels, field_labels, p_traj, p_t, p_xyz, p_val,
             f_dims, f_origin, f_spacing, f_times, f_values):
    """Trajectory split, per-timestep voxel sets and statistics (postproc.py:136-227)."""
    if mmap is None:
        mmap = {r.id: r.id for r in rows}
    members = {}
    for r in rows:
        members.setdefault(mmap[r.id], []).append(r.id)
    feats = {f: FeatureOut(f, sorted(m)) for f, m in members.items()}
    lut = np.full(max([r.id for r in rows] + [0]) + 1, -1, np.int64)
    for i, rep in mmap.items():
        lut[i] = rep
    n_p = len(point_labels)
    if n_p:
        ut = np.unique(p_t)
        stride = np.diff(ut).min() if len(ut) > 1 else np.inf
        fl = lut[np.asarray(point_labels, np.int64)]
        order = np.lexsort((p_t, p_traj))
        tid = p_traj[order]
        cuts = np.flatnonzero(np.r_[True, tid[1:] != tid[:-1]])
        for a, e in zip(cuts, np.r_[cuts[1:], n_p]):
            idx = order[a:e]
            lab, tt = fl[idx], p_t[idx]
            s = 0
            for i in range(1, len(idx) + 1):
                if i < len(idx) and lab[i] == lab[s] and not (tt[i] - tt[i - 1] > stride * (1 + 1e-9)):
                    continue
                run = idx[s:i]
                if len(run) >= 2:
                    feats[int(lab[s])].polylines.append(run)
                else:
                    feats[int(lab[s])].isolated_points.append(int(run[0]))
                s = i
    ncell = int(np.prod(f_dims))
    if len(field_labels):
        fl = lut[np.asarray(field_labels, np.int64)]
        for m in range(len(f_times)):
            lab = fl[m * ncell:(m + 1) * ncell]
            for f in np.unique(lab):
                feats[int(f)].voxels[m] = np.flatnonzero(lab == f)
    out = [feats[f] for f in sorted(feats)]
    cc = cell_centres(f_dims, f_origin, f_spacing) if len(field_labels) else None
    for f in out:
        locs = []
        st = {"p_mean": None, "p_std": None, "f_mean": None, "f_std": None,
              "n_points": 0, "n_fields": 0}
        pidx = np.concatenate([np.concatenate(f.polylines) if f.polylines else np.zeros(0, np.int64),
                               np.asarray(f.isolated_points, np.int64)])
        if len(pidx):
            locs.append(np.column_stack([p_xyz[pidx], p_t[pidx]]))
            v = p_val[pidx]
            st.update(p_mean=float(v.mean()), p_std=float(v.std()), n_points=len(pidx))
        if f.voxels:
            fv = []
            for m, cells in f.voxels.items():
                locs.append(np.column_stack([cc[cells], np.full(len(cells), f_times[m])]))
                fv.append(f_values[m][cells])
                st["n_fields"] += len(cells)
            fv = np.concatenate(fv)
            st.update(f_mean=float(fv.mean()), f_std=float(fv.std()))
        allloc = np.vstack(locs)
        st["bbox_min"] = [float(x) for x in allloc.min(axis=0)]
        st["bbox_max"] = [float(x) for x in allloc.max(axis=0)]
        f.stats = st
    return out
