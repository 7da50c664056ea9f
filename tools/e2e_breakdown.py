"""Phase breakdown of the public assemble() (general strategy) on one
workload: where the end-to-end time goes beyond the device kernels.

    python tools/e2e_breakdown.py [R4]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2101_08825_b200.assembly import AssemblyContext  # noqa: E402
from paper_2101_08825_b200.parallel import pair_counts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "R4"
mesh, space, kp, cfg = bench.build_problem(name)
dev = torch.device("cuda", 0)


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


for trial in range(3):
    t0 = T()
    ctx = AssemblyContext(mesh, space, kp, cfg, dev)
    t1 = T()
    A = ctx.new_matrix()
    t2 = T()
    w = pair_counts(mesh, kp, ctx.dmesh)
    t3 = T()
    cnt = ctx.run_streamed(A)
    t4 = time.perf_counter()          # launches queued, copies running
    ctx.finish(A, cnt)
    t5 = T()
    print(f"  kernels+finish ended at {t5:.3f}", flush=True)
    ctx.join_streamed(A)
    t6 = T()
    print(f"{name} trial {trial}: context+upload {t1 - t0:.3f}s, "
          f"new_matrix {t2 - t1:.3f}s, pair_counts(extra) {t3 - t2:.3f}s, "
          f"run_streamed(host) {t4 - t3:.3f}s, kernels+finish {t5 - t4:.3f}s,"
          f" tail copy {t6 - t5:.3f}s, total(excl. extra) "
          f"{t6 - t0 - (t3 - t2):.3f}s", flush=True)
    del A, ctx
