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
