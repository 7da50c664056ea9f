"""Where a bench step's time goes (device-resident inputs): run / finish
split with host timers around synchronisations.

    python tools/step_breakdown.py [R2-small]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2101_08825_b200 import _native as N  # noqa: E402
from paper_2101_08825_b200.assembly import AssemblyContext  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "R2-small"
mesh, space, kp, cfg = bench.build_problem(name)
dev = torch.device("cuda", 0)
ctx = AssemblyContext(mesh, space, kp, cfg, dev)
A = ctx.new_matrix()
plan = ctx.default_plan()
cnt = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64, device=dev)


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


for trial in range(4):
    t0 = T()
    A._dvals.zero_()
    cnt.zero_()
    t1 = T()
    ctx.run(A, plan=plan, counters=cnt)
    t2 = time.perf_counter()
    t3 = T()
    import ctypes
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    N.check(N.lib().mf_asymmetry_inf(ctypes.byref(A._pattern_struct()),
                                     N.ptr(A._dvals), N.ptr(out),
                                     N.stream_ptr()), "asym")
    t4 = T()
    ctx.finish(A, cnt)
    t5 = T()
    print(f"{name} trial {trial}: zero {t1 - t0:.4f}s run-enqueue "
          f"{t2 - t1:.4f}s run-total {t3 - t1:.4f}s asym {t4 - t3:.4f}s "
          f"finish {t5 - t4:.4f}s", flush=True)
