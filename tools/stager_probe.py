"""Host-side rates on the GPU box: prefault (fill), pinned->pageable copy,
and HostStager D2H of a device array into a fresh host array.

    python tools/stager_probe.py [GB]
"""
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2101_08825_b200.device import HostStager  # noqa: E402

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
n = int(gb * 2**30 / 8)
dev = torch.device("cuda", 0)
src = torch.ones(n, dtype=torch.float64, device=dev)
st = HostStager(dev)
import os  # noqa: E402
print("cpus", os.cpu_count())

host = np.empty(n)
t = time.perf_counter()
st.prefault(host)
t1 = time.perf_counter() - t
print(f"prefault {gb:.1f} GB: {t1:.3f}s = {gb / t1:.1f} GB/s", flush=True)
t = time.perf_counter()
host.fill(1.0)
t2 = time.perf_counter() - t
print(f"fill (mapped, 1 thread): {gb / t2:.1f} GB/s", flush=True)
a = np.ones(n)
step = n // 16
t = time.perf_counter()
with ThreadPoolExecutor(16) as p:
    list(p.map(lambda j: np.copyto(host[j * step:(j + 1) * step],
                                   a[j * step:(j + 1) * step]), range(16)))
t3 = time.perf_counter() - t
print(f"copyto 16 threads (mapped): {gb / t3:.1f} GB/s", flush=True)
for pf in (False, True):
    h = np.empty(n)
    torch.cuda.synchronize()
    t = time.perf_counter()
    if pf:
        st.prefault(h)
    ev = torch.cuda.Event()
    ev.record()
    st.run(src, h, [(ev, 0, n)])
    t4 = time.perf_counter() - t
    assert h[0] == 1.0 and h[-1] == 1.0
    print(f"HostStager D2H fresh array (prefault={pf}): {t4:.3f}s = "
          f"{gb / t4:.1f} GB/s", flush=True)
t = time.perf_counter()
buf = torch.empty(n, dtype=torch.float64, pin_memory=True)
t5 = time.perf_counter() - t
t = time.perf_counter()
buf.copy_(src)
torch.cuda.synchronize()
t6 = time.perf_counter() - t
print(f"pinned alloc {t5:.3f}s, raw D2H into pinned {gb / t6:.1f} GB/s",
      flush=True)
