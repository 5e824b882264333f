"""Numpy mirror of the device synthetic generator (paper_1903_12294_b200/csrc/synth.cu)
— TEST INFRASTRUCTURE ONLY.

Reproduces any sub-block of the benchmark inputs bit for bit (same integer
hash, same IEEE operation order), so parity checks and the CPU baseline can
run on exactly the data the GPU segments.
"""

from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def _h3(seed, a, b):
    with np.errstate(over="ignore"):
        return _mix64(_mix64(np.uint64(seed) ^ _mix64(np.asarray(a, np.uint64))) +
                      np.asarray(b, np.uint64))


def _u01(h):
    return (np.asarray(h, np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def blobs(dims, nt, seed, n_blobs):
    nx, ny, nz = (float(d) for d in dims)
    ntm = float(nt - 1 if nt > 1 else 1)
    n = min(int(n_blobs), 16)
    out = []
    for b in range(n):
        u = [float(_u01(_h3(seed, 1000 + b, q))) for q in range(9)]
        o = {}
        o["cx"] = nx * (0.2 + 0.6 * u[0])
        o["cy"] = ny * (0.2 + 0.6 * u[1])
        o["cz"] = nz * (0.2 + 0.6 * u[2])
        o["rx"] = nx * (0.06 + 0.08 * u[3])
        o["ry"] = ny * (0.06 + 0.08 * u[4])
        o["rz"] = nz * (0.06 + 0.08 * u[5])
        o["vx"] = ((nx * (u[6] - 0.5)) * 0.3) / ntm
        o["vy"] = ((ny * (u[7] - 0.5)) * 0.3) / ntm
        o["vz"] = ((nz * (u[8] - 0.5)) * 0.3) / ntm
        o["fv"] = float(b + 1) / float(n + 1)
        o["pv"] = 1.0 - o["fv"]
        out.append(o)
    return out


def _blob_at(B, x, y, z, m):
    lab = np.full(np.shape(x), -1, np.int64)
    for b, o in enumerate(B):
        dx = (x - (o["cx"] + o["vx"] * m)) / o["rx"]
        dy = (y - (o["cy"] + o["vy"] * m)) / o["ry"]
        dz = (z - (o["cz"] + o["vz"] * m)) / o["rz"]
        inside = (dx * dx + dy * dy + dz * dz) <= 1.0
        lab = np.where((lab < 0) & inside, b, lab)
    return lab


def _noisy(base, seed, idx, noise, dyadic):
    idx = np.asarray(idx, np.uint64)
    u = ((_u01(_h3(seed, idx, 1)) + _u01(_h3(seed, idx, 2))) + _u01(_h3(seed, idx, 3))) + \
        _u01(_h3(seed, idx, 4))
    v = base + noise * (u - 2.0)
    if dyadic:
        v = np.floor(v * 1048576.0) / 1048576.0
        v = np.minimum(np.maximum(v, 0.0), 1.0)
    return v


def field(dims, nt, seed=0, noise=0.05, n_blobs=6, dyadic=False, steps=None, cells=None):
    """(len(steps), len(cells)) values of the requested timesteps and flat cell
    indices (default: all)."""
    nx, ny, nz = (int(d) for d in dims)
    ncell = nx * ny * nz
    B = blobs(dims, nt, seed, n_blobs)
    steps = range(nt) if steps is None else steps
    flat = np.arange(ncell) if cells is None else np.asarray(cells, np.int64)
    x = (flat % nx).astype(float) + 0.5
    y = ((flat // nx) % ny).astype(float) + 0.5
    z = (flat // (nx * ny)).astype(float) + 0.5
    out = np.empty((len(steps), len(flat)))
    fv = np.array([o["fv"] for o in B] + [0.0])
    for r, m in enumerate(steps):
        lab = _blob_at(B, x, y, z, float(m))
        base = fv[lab]                          # lab == -1 -> 0.0 (last entry)
        q = np.uint64(m) * np.uint64(ncell) + flat.astype(np.uint64)
        v = _noisy(base, seed, q, noise, dyadic)
        if dyadic and m == 0:
            v = np.where(flat < 2, flat.astype(float), v)
        out[r] = v
    return out


def points(dims, nt, n_traj, seed=0, noise=0.05, n_blobs=6, dyadic=False, traj=None):
    """(traj_id, t, xyz, value) for the requested trajectories (default: all)."""
    nx, ny, nz = (float(d) for d in dims)
    B = blobs(dims, nt, seed, n_blobs)
    traj = np.arange(n_traj) if traj is None else np.asarray(traj)
    p = np.repeat(traj.astype(np.uint64), nt)
    m = np.tile(np.arange(nt), len(traj)).astype(float)
    q = p * np.uint64(nt) + m.astype(np.uint64)
    sp = np.uint64(seed) ^ np.uint64(0x5bd1e995)
    x0, y0, z0 = nx * _u01(_h3(sp, p, 11)), ny * _u01(_h3(sp, p, 12)), nz * _u01(_h3(sp, p, 13))
    vx = 2.0 * _u01(_h3(sp, p, 14)) - 1.0
    vy = 2.0 * _u01(_h3(sp, p, 15)) - 1.0
    vz = 2.0 * _u01(_h3(sp, p, 16)) - 1.0
    x = np.minimum(np.maximum(x0 + vx * m, 0.0), nx - 2.0 ** -16)
    y = np.minimum(np.maximum(y0 + vy * m, 0.0), ny - 2.0 ** -16)
    z = np.minimum(np.maximum(z0 + vz * m, 0.0), nz - 2.0 ** -16)
    if dyadic:
        x = np.floor(x * 65536.0) / 65536.0
        y = np.floor(y * 65536.0) / 65536.0
        z = np.floor(z * 65536.0) / 65536.0
    lab = _blob_at(B, x, y, z, m)
    pv = np.array([o["pv"] for o in B] + [0.0])
    v = _noisy(pv[lab], sp, q, noise, dyadic)
    if dyadic:
        v = np.where(q < 2, q.astype(float), v)
    return p.astype(np.int64), m, np.column_stack([x, y, z]), v


def taxi_points(dims, nt, n_traj, steps=8, skew=0.7, road_frac=0.02, seed=0, noise=0.05,
                n_blobs=6, traj=None):
    """(traj_id, t, xyz, value) of the taxi-like generator (csrc/synth.cu
    k_synth_taxi) for the requested trajectories (default: all)."""
    nx, ny, nz = (float(d) for d in dims)
    B = blobs(dims, nt, seed, n_blobs)
    traj = np.arange(n_traj) if traj is None else np.asarray(traj)
    n_rows = max(int(road_frac * ny), 1)
    n_cols = max(int(road_frac * nx), 1)
    span = max(nt - steps + 1, 1)
    p = np.repeat(traj.astype(np.uint64), steps)
    j = np.tile(np.arange(steps), len(traj)).astype(float)
    sp = np.uint64(seed) ^ np.uint64(0x7a3c5e91)
    s0 = np.minimum((_u01(_h3(sp, p, 21)) * span).astype(np.int64), span - 1)
    m = s0 + j.astype(np.int64)
    x0, y0 = nx * _u01(_h3(sp, p, 22)), ny * _u01(_h3(sp, p, 23))
    vx = 2.0 * _u01(_h3(sp, p, 24)) - 1.0
    vy = 2.0 * _u01(_h3(sp, p, 25)) - 1.0
    sk = _u01(_h3(sp, p, 26)) < skew
    r = _u01(_h3(sp, p, 27))
    row = _u01(_h3(sp, p, 28)) < 0.5
    qr = np.minimum((r * n_rows).astype(np.int64), n_rows - 1)
    qc = np.minimum((r * n_cols).astype(np.int64), n_cols - 1)
    y_road = np.floor(((qr + 0.5) * ny) / n_rows) + 0.5
    x_road = np.floor(((qc + 0.5) * nx) / n_cols) + 0.5
    on_row, on_col = sk & row, sk & ~row
    y0 = np.where(on_row, y_road, y0)
    vx = np.where(on_row, vx * 3.0, vx)
    vy = np.where(on_row, 0.0, vy)
    x0 = np.where(on_col, x_road, x0)
    vy = np.where(on_col, vy * 3.0, vy)
    vx = np.where(on_col, 0.0, vx)
    x = np.minimum(np.maximum(x0 + vx * j, 0.0), nx - 2.0 ** -16)
    y = np.minimum(np.maximum(y0 + vy * j, 0.0), ny - 2.0 ** -16)
    z = np.full_like(x, 0.5 * nz)
    lab = _blob_at(B, x, y, z, m.astype(float))
    pv = np.array([o["pv"] for o in B] + [0.0])
    q = p * np.uint64(steps) + j.astype(np.uint64)
    v = _noisy(pv[lab], sp, q, noise, False)
    return p.astype(np.int64), m.astype(float), np.column_stack([x, y, z]), v
