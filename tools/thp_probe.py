"""First-touch cost of a fresh 16 GiB host array, plain numpy vs an
anonymous mmap with MADV_HUGEPAGE (GPU box probe for HostStager)."""
import mmap
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
N = 1 << 31  # doubles (16 GiB)


def touch(host, threads=16, chunk=1 << 24):
    def f(a):
        host[a:a + chunk].fill(0.0)
    t = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(f, range(0, host.shape[0], chunk)))
    return time.perf_counter() - t


for rep in range(2):
    a = np.empty(N, dtype=np.float64)
    print("numpy.empty first touch", round(touch(a), 3), "s; again",
          round(touch(a), 3))
    del a
    m = mmap.mmap(-1, N * 8)
    m.madvise(mmap.MADV_HUGEPAGE)
    b = np.frombuffer(m, dtype=np.float64)
    print("mmap+MADV_HUGEPAGE first touch", round(touch(b), 3), "s; again",
          round(touch(b), 3))
    del b, m
