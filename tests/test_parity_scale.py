"""Parity of the CUDA path against the C oracle at the sizes the bench runs.

The oracle (oracle/mfseg_oracle.c, a line-by-line restatement of engine.py,
pinned to the reference's golden vectors by test_oracle_golden.py) is the
checker.  Three kinds of evidence:

* full configs[0] runs (64^3 x 8 field, 100k trajectories x 8 steps,
  k=(8,8,8,4), eps_c=1e-12, 10 iterations): labels array_equal, iteration
  count equal, centres within 1e-12 relative (continuous data: the GPU sums
  exactly, numpy sequentially) and bit-identical on the dyadic family where
  every sum is exact in both;
* windowed spot checks at the configs[1] geometry (256^3 x 32, 2M x 32,
  k=(16,16,16,8)) and at the configs[2] slab geometry (512^3 x 8 steps of the
  64-step box, k=(16,16,16,16)): for passes p in {1, 5, 10} the labels the GPU
  run produced in pass p (with block/brick reuse active) are compared with the
  oracle's assignment given the centres the GPU used in that pass, on whole
  sample-bin blocks (the field kernel's 16^3 x 4 blocks, the point kernel's
  bin-sorted chunks) chosen among the most crowded bins, plus a uniform random
  sample of the whole box;
* a case with large absolute coordinates (origin 1e6, times in Unix seconds);
* the configs[4] slab geometry (1024 x 1024 x 128 planes x 16 steps) and the
  thin configs[3] geometry (one z plane: the field kernels block along time),
  plus full thin-field runs.

Bars: labels bit-exact; centres 1e-12 relative (north_star: 1e-5).
"""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


def _gen(dims, nt, ntraj, seed, dyadic, n_blobs=6, noise=0.05):
    from paper_1903_12294_b200.ingest import synthetic_device
    return synthetic_device(dims, nt, ntraj, seed=seed, noise=noise, n_blobs=n_blobs, dyadic=dyadic)


def _host(t):
    return t.cpu().numpy()


def _state_arrays(st):
    from paper_1903_12294_b200.engine import CenterState
    return CenterState.from_device(st)


def _close(got, want, rtol):
    got, want = np.asarray(got, float), np.asarray(want, float)
    nan = np.isnan(got) & np.isnan(want)
    ok = nan | (np.abs(got - want) <= rtol * np.maximum(np.abs(want), 1.0))
    assert ok.all(), (np.flatnonzero(~ok)[:5], got[~ok][:5], want[~ok][:5])


# ------------------------------------------------------------------ configs[0], full runs

@pytest.mark.parametrize("dyadic,seed", [(False, 0), (True, 1)])
def test_configs0_full_run_vs_oracle(dyadic, seed):
    from oracle import c_oracle
    from paper_1903_12294_b200 import ClusterParams
    from paper_1903_12294_b200.engine import run_device
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
    dims, nt, ntraj = (64, 64, 64), 8, 100_000
    fld, pts, _ = _gen(dims, nt, ntraj, seed, dyadic)
    params = ClusterParams(k=(8, 8, 8, 4), eps_c=1e-12, max_iterations=10)
    normalize_device(pts, fld, params.normalize)
    ext = domain_extent_device(pts, fld)
    prog = []
    r = run_device(pts, fld, ext, params, progress=lambda i, d: prog.append((i, d)))
    ploc = np.column_stack([_host(pts.xyz), _host(pts.t)])
    ref = c_oracle.run_grid(ploc, _host(pts.value), dims, fld.origin, fld.spacing, _host(fld.times),
                            _host(fld.values), ext.mins, ext.maxs, params.k, c_f=params.c_f,
                            w_d=params.w_d, w_p=params.w_p, w_f=params.w_f, eps_c=params.eps_c,
                            max_iterations=params.max_iterations, threads=THREADS)
    np.testing.assert_array_equal(_host(r.field_labels), ref["field_labels"])
    np.testing.assert_array_equal(_host(r.point_labels), ref["point_labels"])
    assert r.iterations_used == ref["iterations_used"] and r.converged == ref["converged"]
    assert [i for i, _ in prog] == list(range(1, ref["iterations_used"] + 1))
    st = _state_arrays(r.state)
    for f in ("n_points", "n_fields", "has_p", "has_f", "dormant"):
        np.testing.assert_array_equal(getattr(st, f), ref[f], err_msg=f)
    if dyadic:   # every sum exact in both -> bit-identical centres and deltas
        np.testing.assert_array_equal(st.loc, ref["loc"])
        np.testing.assert_array_equal(st.pval, ref["pval"])
        np.testing.assert_array_equal(st.fval, ref["fval"])
        np.testing.assert_array_equal([d for _, d in prog], ref["progress"])
    else:
        _close(st.loc, ref["loc"], 1e-12)
        _close(st.pval, ref["pval"], 1e-12)
        _close(st.fval, ref["fval"], 1e-12)


# ------------------------------------------------------------------ windowed checks at scale

def _bins_of(loc, mins, C, k):
    b = np.floor((loc - mins) / C)
    return np.clip(b, 0, np.asarray(k) - 1).astype(np.int64)


def _crowded_bins(cloc, mins, C, k, n, rng):
    """The n sample bins with the most centres in their 3^4 neighbourhood, plus
    n random ones."""
    k = np.asarray(k)
    cb = _bins_of(cloc, mins, C, k)
    cnt = np.zeros(tuple(k[::-1]), np.int64)          # [t][z][y][x]
    np.add.at(cnt, (cb[:, 3], cb[:, 2], cb[:, 1], cb[:, 0]), 1)
    pad = np.pad(cnt, 1)
    nb = np.zeros_like(cnt)
    for dt in range(3):
        for dz in range(3):
            for dy in range(3):
                for dx in range(3):
                    nb += pad[dt:dt + k[3], dz:dz + k[2], dy:dy + k[1], dx:dx + k[0]]
    flat = nb.ravel()
    top = np.argsort(-flat, kind="stable")[:n]
    rnd = rng.choice(flat.size, n, replace=False)
    sel = np.unique(np.concatenate([top, rnd]))
    t, r = np.divmod(sel, k[2] * k[1] * k[0])
    z, r = np.divmod(r, k[1] * k[0])
    y, x = np.divmod(r, k[0])
    return np.column_stack([x, y, z, t]), int(flat[top[0]])


def _field_cells_in_bins(bins, dims, origin, spacing, times, mins, C, k):
    """Flat indices of every field cell whose sample bin is one of `bins`."""
    axes = []
    for d in range(3):
        c = origin[d] + (np.arange(dims[d]) + 0.5) * spacing[d]
        axes.append(_bins_of(c[:, None], mins[d:d + 1], C[d:d + 1], k[d:d + 1])[:, 0])
    tb = _bins_of(np.asarray(times)[:, None], mins[3:], C[3:], k[3:])[:, 0]
    ncell = int(np.prod(dims))
    out = []
    for b in bins:
        ii, jj, kk, mm = (np.flatnonzero(axes[0] == b[0]), np.flatnonzero(axes[1] == b[1]),
                          np.flatnonzero(axes[2] == b[2]), np.flatnonzero(tb == b[3]))
        if min(len(ii), len(jj), len(kk), len(mm)) == 0:
            continue
        cell = (ii[None, None, :] + dims[0] * (jj[None, :, None] + dims[1] * kk[:, None, None])).ravel()
        out.append((mm[:, None] * ncell + cell[None, :]).ravel())
    return np.unique(np.concatenate(out)) if out else np.zeros(0, np.int64)


def _with_iters(params, m):
    """params with max_iterations = m (m = 0 allowed: the run stops after the
    initial pass; ClusterParams itself requires >= 1)."""
    from types import SimpleNamespace
    d = params.to_dict()
    d["k"], d["max_iterations"] = tuple(params.k), m
    return SimpleNamespace(**d)


def _windowed(dims, nt, ntraj, k, seed, passes, n_bins=8, n_random=1_000_000, origin=None,
              times=None, xyz_shift=None, w=None):
    from oracle import c_oracle
    from paper_1903_12294_b200 import ClusterParams
    from paper_1903_12294_b200.engine import DeviceField, run_device
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
    from paper_1903_12294_b200.model import interval_distances
    fld, pts, _ = _gen(dims, nt, ntraj, seed, False)
    if origin is not None:     # large absolute coordinates: shift the whole box
        fld = DeviceField(fld.dims, np.asarray(origin, float), fld.spacing,
                          torch.as_tensor(times, dtype=torch.float64, device=fld.values.device),
                          fld.values)
        pts.xyz += torch.as_tensor(xyz_shift, dtype=torch.float64, device=pts.xyz.device)
        tmap = torch.as_tensor(times, dtype=torch.float64, device=pts.t.device)
        pts.t.copy_(tmap[pts.t.long()])
    params = ClusterParams(k=k, eps_c=1e-12, max_iterations=max(passes), **(w or {}))
    normalize_device(pts, fld, True)
    ext = domain_extent_device(pts, fld)
    C = interval_distances(ext, k)
    fvals, ftimes = _host(fld.values), _host(fld.times)
    ploc = np.column_stack([_host(pts.xyz), _host(pts.t)])
    pval = _host(pts.value)
    rng = np.random.default_rng(seed)
    checked = {"field": 0, "point": 0}
    for p in passes:
        # centres used by pass p = final state of the run that stopped after pass p-1
        prev = run_device(pts, fld, ext, _with_iters(params, p - 1))
        cs = _state_arrays(prev.state)
        cur = run_device(pts, fld, ext, _with_iters(params, p))
        assert prev.iterations_used == p - 1 and cur.iterations_used == p
        gfl, gpl = _host(cur.field_labels), _host(cur.point_labels)
        bins, crowd = _crowded_bins(cs.loc, ext.mins, C, k, n_bins, rng)
        fidx = _field_cells_in_bins(bins, dims, fld.origin, fld.spacing, ftimes, ext.mins, C, k)
        fidx = np.unique(np.concatenate([fidx, rng.choice(gfl.size, min(n_random, gfl.size),
                                                          replace=False)]))
        want = c_oracle.assign_field(dims, fld.origin, fld.spacing, ftimes, fvals, cs.loc, cs.fval,
                                     cs.has_f, ext.mins, C, k, params.w_f, params.w_d, params.c_f,
                                     idx=fidx, threads=THREADS)
        bad = np.flatnonzero(gfl[fidx] != want)
        assert bad.size == 0, (p, "field", fidx[bad[:5]], gfl[fidx[bad[:5]]], want[bad[:5]])
        pb = _bins_of(ploc, ext.mins, C, k)
        in_bins = np.zeros(len(ploc), bool)
        key = ((pb[:, 3] * k[2] + pb[:, 2]) * k[1] + pb[:, 1]) * k[0] + pb[:, 0]
        bkey = ((bins[:, 3] * k[2] + bins[:, 2]) * k[1] + bins[:, 1]) * k[0] + bins[:, 0]
        in_bins |= np.isin(key, bkey)
        in_bins[rng.choice(len(ploc), min(n_random // 4, len(ploc)), replace=False)] = True
        pidx = np.flatnonzero(in_bins)
        want = c_oracle.assign(ploc[pidx], pval[pidx], cs.loc, cs.pval, cs.has_p, ext.mins, C, k,
                               params.w_p, params.w_d, params.c_f, threads=THREADS)
        bad = np.flatnonzero(gpl[pidx] != want)
        assert bad.size == 0, (p, "point", pidx[bad[:5]], gpl[pidx[bad[:5]]], want[bad[:5]])
        checked["field"] += fidx.size
        checked["point"] += pidx.size
        assert crowd > 0
    return checked


def test_configs1_windows_vs_oracle():
    """configs[1] geometry: 256^3 x 32, 2M trajectories x 32 steps, k=(16,16,16,8)."""
    got = _windowed((256, 256, 256), 32, 2_000_000, (16, 16, 16, 8), 3, passes=(1, 5, 10))
    assert got["field"] > 3 * 1_000_000 and got["point"] > 3 * 250_000


def test_configs2_slab_windows_vs_oracle():
    """configs[2] per-GPU slab geometry: 512^3 x 8 steps, 16M trajectories,
    k=(16,16,16,2) over the slab (cells 32 voxels wide, 4 timesteps deep)."""
    got = _windowed((512, 512, 512), 8, 16_000_000, (16, 16, 16, 2), 4, passes=(1, 5))
    assert got["field"] > 2 * 1_000_000


def test_large_absolute_coordinates_vs_oracle():
    """Origin at 1e6, times in Unix seconds (1-minute steps): the fp32 screens'
    chunk-relative coordinates and the fixed-point sums must stay exact."""
    nt = 12
    times = 1.7e9 + 60.0 * np.arange(nt)
    got = _windowed((96, 80, 64), nt, 40_000, (6, 5, 4, 3), 6, passes=(1, 4),
                    origin=(1e6, -2e6, 3.5e5), times=times, xyz_shift=(1e6, -2e6, 3.5e5),
                    w=dict(c_f=1e-3))
    assert got["field"] > 0 and got["point"] > 0


# ------------------------------------------------------------------ thin (2-D + time) fields

@pytest.mark.parametrize("c_f,seed", [(1.0, 7), (0.6, 8)])
def test_thin_field_full_run_vs_oracle(c_f, seed):
    """A field of one z plane (the configs[3] shape, k_z = 1): the field kernels
    run their z axis over the timesteps (FieldArgs.swap_zt).  Full run against
    the C oracle: labels array_equal, centres within 1e-12."""
    from oracle import c_oracle
    from paper_1903_12294_b200 import ClusterParams
    from paper_1903_12294_b200.engine import run_device
    from paper_1903_12294_b200.ingest import domain_extent_device, normalize_device
    dims, nt, ntraj = (96, 80, 1), 40, 30_000
    fld, pts, _ = _gen(dims, nt, ntraj, seed, False)
    params = ClusterParams(k=(6, 5, 1, 7), eps_c=1e-12, max_iterations=6, c_f=c_f)
    normalize_device(pts, fld, params.normalize)
    ext = domain_extent_device(pts, fld)
    r = run_device(pts, fld, ext, params)
    ploc = np.column_stack([_host(pts.xyz), _host(pts.t)])
    ref = c_oracle.run_grid(ploc, _host(pts.value), dims, fld.origin, fld.spacing, _host(fld.times),
                            _host(fld.values), ext.mins, ext.maxs, params.k, c_f=params.c_f,
                            w_d=params.w_d, w_p=params.w_p, w_f=params.w_f, eps_c=params.eps_c,
                            max_iterations=params.max_iterations, threads=THREADS)
    np.testing.assert_array_equal(_host(r.field_labels), ref["field_labels"])
    np.testing.assert_array_equal(_host(r.point_labels), ref["point_labels"])
    assert r.iterations_used == ref["iterations_used"]
    st = _state_arrays(r.state)
    _close(st.loc, ref["loc"], 1e-12)
    _close(st.fval, ref["fval"], 1e-12)
    _close(st.pval, ref["pval"], 1e-12)


def test_configs3_geometry_windows_vs_oracle():
    """configs[3]-like thin geometry (one z plane, 16-cell x 16-cell x 8-step bins)."""
    got = _windowed((512, 512, 1), 48, 300_000, (32, 32, 1, 6), 9, passes=(1, 4))
    assert got["field"] > 1_000_000 and got["point"] > 0


def test_configs4_slab_geometry_windows_vs_oracle():
    """configs[4] per-GPU slab geometry: 1024 x 1024 x 128 planes x 16 steps,
    k=(32, 32, 4, 4) (bins of 32^3 cells x 4 timesteps), 16M trajectories' worth
    of points in the slab scaled down to 4M."""
    got = _windowed((1024, 1024, 128), 16, 4_000_000, (32, 32, 4, 4), 11, passes=(1, 4),
                    n_bins=6, n_random=1_000_000)
    assert got["field"] > 1_000_000 and got["point"] > 0
