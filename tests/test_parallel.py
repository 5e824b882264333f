"""Multi-rank logic of the time-slab sharding, on CPU with gloo (world size 2).

The data-path collective is a SUM all-reduce of exact 128-bit fixed-point
partial sums exchanged as 42-bit limbs (paper_1903_12294_b200/parallel.py,
csrc/update.cu k_to_limbs / k_from_limbs).  These tests check, with real
torch.distributed processes, that (1) the slab split partitions the timesteps,
(2) global min/max agree exactly, (3) the limb all-reduce reconstructs the
exact total, and (4) per-slab exact partial sums of a sharded assignment add
up to the unsharded sums, so centres are identical for any rank count.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1903_12294_b200.parallel import allreduce_limbs, global_minmax, tbin_slabs, time_slab

M42 = (1 << 42) - 1


def to_limbs(v: int):
    """Python restatement of k_to_limbs: 128-bit two's complement -> 3 limbs."""
    v &= (1 << 128) - 1
    s = v - (1 << 128) if v >> 127 else v
    return [s & M42, (s >> 42) & M42, s >> 84]


def from_limbs(l):
    return l[0] + (l[1] << 42) + (l[2] << 84)


def fix(x: float) -> int:
    """x * 2^64 truncated toward zero (d2fix)."""
    from fractions import Fraction
    f = Fraction(x) * (1 << 64)
    return int(f)      # int() truncates toward zero


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


def test_time_slab_partition():
    for nt in (1, 2, 7, 32, 33):
        for world in (1, 2, 3, 8):
            covered = []
            for r in range(world):
                a, b = time_slab(r, world, nt)
                assert 0 <= a <= b <= nt
                covered.extend(range(a, b))
            assert covered == list(range(nt))


def test_tbin_slabs_whole_bins():
    """Slab boundaries fall on t-bin changes and the slabs partition the steps."""
    for nt, k_t, world in ((32, 8, 2), (64, 16, 4), (256, 64, 8), (33, 8, 3), (7, 2, 4), (10, 1, 2)):
        times = np.arange(nt, dtype=float)
        C_t = (nt - 1.0) / k_t
        slabs = tbin_slabs(times, 0.0, C_t, k_t, world)
        b = np.clip(np.floor(times / C_t), 0, k_t - 1)
        covered = []
        for m0, m1 in slabs:
            covered.extend(range(m0, m1))
            if 0 < m0 < nt and m1 > m0:
                assert b[m0] != b[m0 - 1]           # starts a new t-bin
        assert covered == list(range(nt))
        owners = {}
        for r, (m0, m1) in enumerate(slabs):
            for m in range(m0, m1):
                assert owners.setdefault(b[m], r) == r   # a t-bin lives on one rank
    # the bench's weak-scaling layout: 32 steps per rank, k_t = 8 per rank
    for world in (1, 2, 4, 8):
        nt = 32 * world
        assert tbin_slabs(np.arange(nt, dtype=float), 0.0, (nt - 1.0) / (8 * world), 8 * world,
                          world) == [(32 * r, 32 * r + 32) for r in range(world)]


def _minmax_fn(rank, world):
    vals = [np.array([0.5, 3.25]), np.array([-1.0, 2.0])][rank]
    return global_minmax(float(vals.min()), float(vals.max()))


def test_global_minmax_gloo():
    res = run_ranks(_minmax_fn)
    assert res[0] == res[1] == (-1.0, 3.25)


def _limb_fn(rank, world):
    rng = np.random.default_rng(rank)
    words = [int(x) for x in rng.integers(-2**62, 2**62, 16)]
    words = [w * (1 << 40) + int(rng.integers(0, 2**40)) for w in words]   # ~102-bit values
    limbs = torch.tensor([l for w in words for l in to_limbs(w)], dtype=torch.int64)
    allreduce_limbs(limbs)
    got = [from_limbs(limbs[3 * i:3 * i + 3].tolist()) for i in range(16)]
    return words, got


def test_limb_allreduce_is_exact():
    res = run_ranks(_limb_fn)
    total = [a + b for a, b in zip(res[0][0], res[1][0])]
    for r in range(2):
        assert res[r][1] == total


def _shard_fn(rank, world):
    """Each rank assigns its time slab with the oracle, forms exact fixed-point
    partial sums, and all-reduces them as limbs."""
    from oracle import c_oracle
    from oracle import mfseg_oracle as O
    from oracle import synth
    dims, nt, ntraj, k = (16, 12, 8), 6, 120, (4, 3, 2, 2)
    vals = synth.field(dims, nt, seed=5)
    _, t, xyz, pv = synth.points(dims, nt, ntraj, seed=5)
    mins, maxs = np.zeros(4), np.array([16.0, 12.0, 8.0, nt - 1.0])
    C = O.interval_lengths(mins, maxs, k)
    K = int(np.prod(k))
    seeds = O.seed_locations(mins, C, k)
    cval = np.linspace(0.0, 1.0, K)
    has = np.ones(K, np.uint8)
    m0, m1 = time_slab(rank, world, nt)
    floc = O.field_locations(dims, np.zeros(3), np.ones(3), np.arange(nt, dtype=float))
    ncell = int(np.prod(dims))
    fl_loc, fl_val = floc[m0 * ncell:m1 * ncell], vals[m0:m1].reshape(-1)
    sel = (t >= m0) & (t < m1)
    ploc, pval = np.column_stack([xyz, t])[sel], pv[sel]
    fl = c_oracle.assign(fl_loc, fl_val, seeds, cval, has, mins, C, k, 1.0, 1.0, 1.0, threads=1)
    pl = c_oracle.assign(ploc, pval, seeds, cval, has, mins, C, k, 1.0, 1.0, 1.0, threads=1)
    sums = [[0] * 6 for _ in range(K)]   # x, y, z, t, pv+fv, count
    for lab, loc, v in list(zip(fl, fl_loc, fl_val)) + list(zip(pl, ploc, pval)):
        for d in range(4):
            sums[lab][d] += fix(loc[d])
        sums[lab][4] += fix(v)
        sums[lab][5] += 1
    limbs = torch.tensor([l for row in sums for w in row for l in to_limbs(w)], dtype=torch.int64)
    allreduce_limbs(limbs)
    flat = [from_limbs(limbs[3 * i:3 * i + 3].tolist()) for i in range(K * 6)]
    return flat


def test_sharded_exact_sums_match_single_rank():
    two = run_ranks(_shard_fn, world=2)
    one = run_ranks(_shard_fn, world=1)
    assert two[0] == two[1] == one[0]


# ------------------------------------------------------------------ z-slabs, bin ranges, points

def test_zbin_slabs_and_bin_ranges_partition():
    """z-plane slabs of whole z-bins; the per-rank bin ranges give every point
    exactly one owner (also points outside the field's bins)."""
    from paper_1903_12294_b200.parallel import (bins_of, cell_centres, select_points_for_slab,
                                                slab_bin_ranges, zbin_slabs)
    rng = np.random.default_rng(3)
    for nz, k_z, world, origin, spacing in ((64, 8, 2, 0.0, 1.0), (128, 32, 8, -3.7, 0.31),
                                            (10, 3, 4, 0.0, 1.0), (33, 4, 3, 1e6, 0.125)):
        z_min = origin - 0.01
        C_z = (nz * spacing + 0.02) / k_z
        slabs = zbin_slabs(nz, origin, spacing, z_min, C_z, k_z, world)
        zc = cell_centres(nz, origin, spacing)
        b = bins_of(zc, z_min, C_z, k_z)
        covered = [k for k0, k1 in slabs for k in range(k0, k1)]
        assert covered == list(range(nz))
        for k0, k1 in slabs:
            if 0 < k0 < nz and k1 > k0:
                assert b[k0] != b[k0 - 1]
        ranges = slab_bin_ranges(zc, z_min, C_z, k_z, slabs)
        pz = rng.uniform(z_min - 5 * C_z, z_min + (k_z + 5) * C_z, 5000)
        owners = np.zeros(len(pz), int)
        for r, (b0, b1) in enumerate(ranges):
            owners += select_points_for_slab(pz, z_min, C_z, k_z, b0, b1).astype(int)
            for k0, k1 in [slabs[r]]:
                if k1 > k0:   # the rank's own cells are inside its bin range
                    assert np.all((b[k0:k1] >= b0) & (b[k0:k1] < b1))
        assert np.all(owners == 1)


def _extent_fn(rank, world):
    """normalize_and_extent_sharded (values untouched: normalize off) on CPU
    tensors equals the host extent of the union."""
    from paper_1903_12294_b200.engine import DeviceField, DevicePoints
    from paper_1903_12294_b200.parallel import normalize_and_extent_sharded
    rng = np.random.default_rng(10 + rank)
    n = 50 + 30 * rank
    xyz = torch.as_tensor(rng.uniform(-2, 9, (n, 3)))
    t = torch.as_tensor(rng.uniform(0, 5, n))
    v = torch.as_tensor(rng.normal(size=n))
    nz_local = 3
    fld = DeviceField((4, 5, nz_local), np.array([0.5, -1.0, 2.0]), np.array([0.25, 0.5, 1.0]),
                      torch.arange(3, dtype=torch.float64) * 2.0,
                      torch.as_tensor(rng.normal(size=3 * 4 * 5 * nz_local)), (0, 0, nz_local * rank))
    ext, norm = normalize_and_extent_sharded(DevicePoints(xyz, t, v), fld, False,
                                             grid_dims=(4, 5, nz_local * world))
    return (ext.mins.tolist(), ext.maxs.tolist(), norm.enabled,
            xyz.numpy(), t.numpy())


def test_normalize_and_extent_sharded_gloo():
    res = run_ranks(_extent_fn)
    assert res[0][:3] == res[1][:3]
    xyz = np.vstack([r[3] for r in res])
    t = np.concatenate([r[4] for r in res])
    mins, maxs, enabled = res[0][:3]
    assert enabled is False
    field_lo = np.array([0.5, -1.0, 2.0, 0.0])
    field_hi = np.array([0.5 + 4 * 0.25, -1.0 + 5 * 0.5, 2.0 + 6 * 1.0, 4.0])
    want_lo = np.minimum(field_lo, np.r_[xyz.min(0), t.min()])
    want_hi = np.maximum(field_hi, np.r_[xyz.max(0), t.max()])
    assert mins == want_lo.tolist() and maxs == want_hi.tolist()


def _nonfinite_fn(rank, world):
    from paper_1903_12294_b200.engine import DeviceField, DevicePoints
    from paper_1903_12294_b200.parallel import normalize_and_extent_sharded
    v = torch.tensor([0.0, float("nan") if rank == 1 else 1.0], dtype=torch.float64)
    pts = DevicePoints(torch.zeros((2, 3), dtype=torch.float64), torch.zeros(2, dtype=torch.float64), v)
    fld = DeviceField((1, 1, 1), np.zeros(3), np.ones(3), torch.zeros(0, dtype=torch.float64),
                      torch.zeros(0, dtype=torch.float64))
    try:
        normalize_and_extent_sharded(pts, fld, False)
    except ValueError as e:
        return str(e)
    return None


def test_sharded_non_finite_rejected_on_every_rank():
    res = run_ranks(_nonfinite_fn)
    assert all(r is not None and "non-finite" in r for r in res)


# ------------------------------------------------------------------ sharded feature materialisation

def test_fix128_limb_roundtrip():
    from paper_1903_12294_b200.postproc import fix128_to_limbs, limbs_to_fix128
    rng = np.random.default_rng(0)
    vals = [int(x) * (1 << 50) + int(y) for x, y in zip(rng.integers(-2**62, 2**62, 64),
                                                          rng.integers(0, 2**50, 64))]
    def pair(v):
        u = v & ((1 << 128) - 1)
        lo, hi = u & ((1 << 64) - 1), u >> 64
        return [lo - (1 << 64) if lo >> 63 else lo, hi - (1 << 64) if hi >> 63 else hi]
    w = torch.tensor([pair(v) for v in vals], dtype=torch.int64)
    L = fix128_to_limbs(w)
    assert torch.equal(limbs_to_fix128(L), w)
    # sums of several values through the limbs
    L3 = L[:16] + L[16:32] + L[32:48]
    back = limbs_to_fix128(L3)
    for i in range(16):
        lo, hi = int(back[i, 0]) & ((1 << 64) - 1), int(back[i, 1])
        assert hi * (1 << 64) + lo == vals[i] + vals[16 + i] + vals[32 + i]


def _stat_fn(rank, world):
    from paper_1903_12294_b200.postproc import reduce_stat_partials
    rng = np.random.default_rng(20 + rank)
    n = 5
    S = torch.zeros((n, 18), dtype=torch.int64)
    S[:, 0:8] = torch.as_tensor(rng.integers(-2**40, 2**40, (n, 8)))
    S[:, 1::2][:, :4] = torch.as_tensor(rng.integers(-3, 3, (n, 4)))   # hi words
    S[:, 8:10] = torch.as_tensor(rng.integers(0, 100, (n, 2)))
    keys = rng.integers(-2**63, 2**63 - 1, (n, 8), dtype=np.int64)
    S[:, 10:18] = torch.as_tensor(keys)
    before = S.clone()
    reduce_stat_partials(S)
    return before, S


def test_reduce_stat_partials_gloo():
    res = run_ranks(_stat_fn)
    a, b = res[0][0], res[1][0]
    for r in range(2):
        S = res[r][1]
        for i in range(a.shape[0]):
            for w in range(4):
                def val(T):
                    return int(T[i, 2 * w + 1]) * (1 << 64) + (int(T[i, 2 * w]) & ((1 << 64) - 1))
                assert val(S) == val(a) + val(b)
        assert torch.equal(S[:, 8:10], a[:, 8:10] + b[:, 8:10])
        ua, ub = a[:, 10:18].numpy().view(np.uint64), b[:, 10:18].numpy().view(np.uint64)
        us = S[:, 10:18].numpy().view(np.uint64)
        assert np.array_equal(us[:, :4], np.minimum(ua[:, :4], ub[:, :4]))
        assert np.array_equal(us[:, 4:], np.maximum(ua[:, 4:], ub[:, 4:]))


def _traj_fn(rank, world):
    from paper_1903_12294_b200.postproc import exchange_by_trajectory, global_stride
    rng = np.random.default_rng(30 + rank)
    n = 200 + 50 * rank
    tid = torch.as_tensor(rng.integers(-20, 60, n), dtype=torch.int64)
    t = torch.as_tensor(rng.integers(0, 10, n) * 0.5 + 0.25 * rank)
    gidx = torch.arange(n, dtype=torch.int64) + 1000 * rank
    o_tid, (o_t, o_g) = exchange_by_trajectory(tid, [t, gidx])
    return tid.numpy(), gidx.numpy(), o_tid.numpy(), o_t.numpy(), o_g.numpy(), global_stride(t)


def test_exchange_by_trajectory_gloo():
    res = run_ranks(_traj_fn)
    all_tid = np.concatenate([r[0] for r in res])
    all_g = np.concatenate([r[1] for r in res])
    got_g = np.concatenate([r[4] for r in res])
    assert sorted(got_g.tolist()) == sorted(all_g.tolist())      # every sample once
    owners = {}
    for r, rr in enumerate(res):
        for tr in rr[2].tolist():
            assert owners.setdefault(tr, r) == r                # a trajectory has one owner
        if r and len(rr[2]) and len(res[r - 1][2]):
            assert rr[2].min() > res[r - 1][2].max()            # owner ranges increase with rank
        # every received sample keeps its own (traj, t, index)
        g2t = dict(zip(all_g.tolist(), all_tid.tolist()))
        assert all(g2t[g] == tr for g, tr in zip(rr[4].tolist(), rr[2].tolist()))
    assert res[0][5] == res[1][5] == 0.25
