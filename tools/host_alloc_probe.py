"""Fresh 16.4 GB host array: fault-in strategies and D2H rates (diagnostic)."""
import ctypes, mmap, sys, time, threading
import numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
n = 2053225511
dev = torch.device("cuda", 0)
src = torch.ones(n, dtype=torch.float64, device=dev)
libc = ctypes.CDLL("libc.so.6")
MADV_HUGEPAGE = 14
def T(): torch.cuda.synchronize(); return time.perf_counter()
def touch(a, nthr):
    step = -(-a.size // nthr)
    with ThreadPoolExecutor(nthr) as p:
        list(p.map(lambda k: a[k*step:(k+1)*step].fill(0.0), range(nthr)))
def copy_par(h, nthr):
    ht = torch.from_numpy(h); step = -(-n // nthr)
    streams = [torch.cuda.Stream() for _ in range(nthr)]
    def piece(k):
        with torch.cuda.stream(streams[k]):
            ht[k*step:min(n,(k+1)*step)].copy_(src[k*step:min(n,(k+1)*step)])
    with ThreadPoolExecutor(nthr) as p: list(p.map(piece, range(nthr)))
for huge in (False, True):
    for nthr in (8, 16):
        t = T(); h = np.empty(n)
        if huge:
            addr = h.ctypes.data; off = addr % 4096
            libc.madvise(ctypes.c_void_p(addr - off), ctypes.c_size_t(h.nbytes + off), MADV_HUGEPAGE)
        t1 = T(); touch(h, nthr); t2 = T()
        copy_par(h, 4); t3 = T()
        print(f"huge={huge} touch({nthr} thr) {t2-t1:.3f}s  par-copy(4 streams) {t3-t2:.3f}s ({n*8/(t3-t2)/1e9:.1f} GB/s)  total {t3-t:.3f}s", flush=True)
        del h
# copies into fresh memory directly with parallel streams (faults inside copy)
for nthr in (4, 8):
    t = T(); h = np.empty(n); copy_par(h, nthr); t2 = T()
    print(f"fresh par-copy {nthr} streams: {t2-t:.3f}s ({n*8/(t2-t)/1e9:.1f} GB/s)", flush=True)
    del h
