"""D2H staging rate while a long kernel runs (is the copy starved?).

Launches ~3 s of mf_fp64_probe on the compute stream, then stages an 8 GB
device array to a fresh host array with HostStager while the main thread
waits in (a) torch .cpu() of a scalar, (b) Event.synchronize(), (c) a
time.sleep polling loop.
"""
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2101_08825_b200 import _native as N  # noqa: E402
from paper_2101_08825_b200.device import HostStager  # noqa: E402

dev = torch.device("cuda", 0)
n = 2**30  # 8 GB
src = torch.ones(n, dtype=torch.float64, device=dev)
out = torch.zeros(1, dtype=torch.float64, device=dev)
st = HostStager(dev)
L = N.lib()


def busy(iters):
    N.check(L.mf_fp64_probe(N.ptr(out), iters, 148 * 8, 256,
                            N.stream_ptr()), "probe")


busy(1000)
torch.cuda.synchronize()
t = time.perf_counter()
busy(200000)
torch.cuda.synchronize()
per = (time.perf_counter() - t) / 200000
iters = int(3.0 / per)
for mode in ("cpu", "event", "sleep"):
    host = np.empty(n)
    st.prefault(host)
    ev = torch.cuda.Event()
    ev.record()
    busy(iters)
    done_evt = torch.cuda.Event()
    done_evt.record()
    t0 = time.perf_counter()
    res = {}

    def worker():
        st.run(src, host, [(ev, 0, n)])
        res["t"] = time.perf_counter() - t0

    th = threading.Thread(target=worker)
    th.start()
    if mode == "cpu":
        _ = out.cpu()
    elif mode == "event":
        done_evt.synchronize()
    else:
        while not done_evt.query():
            time.sleep(0.001)
    tk = time.perf_counter() - t0
    th.join()
    print(f"main waits via {mode}: kernel done {tk:.2f}s, 8 GB staged "
          f"{res['t']:.2f}s", flush=True)
