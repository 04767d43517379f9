"""Host<->device transfer rates on the GPU box (pageable / pinned, 2 GB)."""
import time

import numpy as np
import torch

dev = torch.device("cuda", 0)
nb = 2 * 1024**3
a = np.ones(nb // 8)
t = torch.empty(nb // 8, dtype=torch.float64, device=dev)
torch.cuda.synchronize()


def tm(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def gbs(s):
    return f"{s * 1e3:.1f} ms = {nb / s / 1e9:.1f} GB/s"


print("pageable H2D (torch.from_numpy.to):", gbs(tm(lambda: t.copy_(torch.from_numpy(a)))))
print("pageable D2H:", gbs(tm(lambda: torch.from_numpy(a).copy_(t))))
t0 = time.perf_counter()
p = torch.empty(nb // 8, dtype=torch.float64, pin_memory=True)
print(f"pinned alloc 2 GB: {1e3 * (time.perf_counter() - t0):.1f} ms")
pn = p.numpy()
print("pinned H2D:", gbs(tm(lambda: t.copy_(p, non_blocking=True))))
print("pinned D2H:", gbs(tm(lambda: p.copy_(t, non_blocking=True))))
print("host memcpy pageable->pinned (np.copyto):", gbs(tm(lambda: np.copyto(pn, a))))
b = np.empty_like(a)
print("host memcpy pageable->pageable:", gbs(tm(lambda: np.copyto(b, a))))
import concurrent.futures as cf

ex = cf.ThreadPoolExecutor(8)


def par_copy(dst, src, k=8):
    n = src.size
    fs = [ex.submit(np.copyto, dst[i * n // k:(i + 1) * n // k], src[i * n // k:(i + 1) * n // k]) for i in range(k)]
    for f in fs:
        f.result()


print("host memcpy 8 threads pageable->pinned:", gbs(tm(lambda: par_copy(pn, a))))
del p
t0 = time.perf_counter()
p2 = torch.empty(nb // 8, dtype=torch.float64, pin_memory=True)
print(f"pinned alloc again (caching allocator): {1e3 * (time.perf_counter() - t0):.1f} ms")
import os
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
