"""Host<->device copy rates for the e2e design: pinned vs pageable vs
cudaHostRegister'ed numpy buffers, whole-array and chunked, plus f32 uploads."""
import time

import numpy as np
import torch

N = 1 << 29          # 512M doubles = 4.3 GB (the c2 field)
dev = torch.device("cuda", 0)
d = torch.empty(N, dtype=torch.float64, device=dev)


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


def rate(nbytes, f, reps=3):
    best = 1e9
    for _ in range(reps):
        t0 = T()
        f()
        best = min(best, T() - t0)
    return nbytes / best / 1e9, best


a = np.random.default_rng(0).random(N)          # pageable
p = torch.empty(N, dtype=torch.float64, pin_memory=True)
p.copy_(torch.from_numpy(a))
print(f"pinned H2D    {rate(8 * N, lambda: d.copy_(p, non_blocking=True))[0]:.1f} GB/s", flush=True)
print(f"pageable H2D  {rate(8 * N, lambda: d.copy_(torch.from_numpy(a)))[0]:.1f} GB/s", flush=True)
print(f"pinned D2H    {rate(8 * N, lambda: p.copy_(d, non_blocking=True))[0]:.1f} GB/s", flush=True)
print(f"pageable D2H  {rate(8 * N, lambda: torch.from_numpy(a).copy_(d))[0]:.1f} GB/s", flush=True)

cr = torch.cuda.cudart()
t0 = time.perf_counter()
rc = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
t1 = time.perf_counter()
print(f"cudaHostRegister 4.3 GB: rc={rc} {1e3 * (t1 - t0):.1f} ms", flush=True)
print(f"registered H2D {rate(8 * N, lambda: d.copy_(torch.from_numpy(a), non_blocking=True))[0]:.1f} GB/s",
      flush=True)
t0 = time.perf_counter()
cr.cudaHostUnregister(a.ctypes.data)
print(f"cudaHostUnregister: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)

# chunked pageable -> pinned ring -> device, host copies on 4 threads
from concurrent.futures import ThreadPoolExecutor
CH = 1 << 24          # 128 MB chunks
ring = [torch.empty(CH, dtype=torch.float64, pin_memory=True) for _ in range(4)]
evs = [torch.cuda.Event() for _ in ring]
cs = torch.cuda.Stream()
pool = ThreadPoolExecutor(8)


def staged():
    src = torch.from_numpy(a)
    nch = N // CH
    futs = {}
    for i in range(min(4, nch)):
        futs[i] = pool.submit(ring[i].copy_, src[i * CH:(i + 1) * CH])
    for i in range(nch):
        futs.pop(i).result()
        b = ring[i % 4]
        with torch.cuda.stream(cs):
            d[i * CH:(i + 1) * CH].copy_(b, non_blocking=True)
            evs[i % 4].record(cs)
        if i + 4 < nch:
            evs[i % 4].synchronize()
            futs[i + 4] = pool.submit(ring[i % 4].copy_, src[(i + 4) * CH:(i + 5) * CH])
    cs.synchronize()


print(f"staged pageable H2D (4 x 128 MB ring) {rate(8 * N, staged)[0]:.1f} GB/s", flush=True)

f = a.astype(np.float32)
pf = torch.empty(N, dtype=torch.float32, pin_memory=True)
pf.copy_(torch.from_numpy(f))
df = torch.empty(N, dtype=torch.float32, device=dev)
print(f"pinned f32 H2D {rate(4 * N, lambda: df.copy_(pf, non_blocking=True))[0]:.1f} GB/s (bytes)",
      flush=True)
i32 = torch.empty(N, dtype=torch.int32, device=dev)
pi = torch.empty(N, dtype=torch.int32, pin_memory=True)
print(f"pinned int32 D2H {rate(4 * N, lambda: pi.copy_(i32, non_blocking=True))[0]:.1f} GB/s",
      flush=True)
# simultaneous H2D + D2H (full duplex?)
s2 = torch.cuda.Stream()


def duplex():
    with torch.cuda.stream(cs):
        d.copy_(p, non_blocking=True)
    with torch.cuda.stream(s2):
        pi.copy_(i32, non_blocking=True)
    cs.synchronize()
    s2.synchronize()


r, t = rate(8 * N + 4 * N, duplex)
print(f"duplex H2D 4.3 GB + D2H 2.1 GB: {1e3 * t:.1f} ms ({r:.1f} GB/s combined)", flush=True)
