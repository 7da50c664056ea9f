"""One general-path assembly of a workload (for ncu captures)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2101_08825_b200 import _native as N  # noqa: E402
from paper_2101_08825_b200.assembly import AssemblyContext  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "R4-small"
mesh, space, kp, cfg = bench.build_problem(name)
ctx = AssemblyContext(mesh, space, kp, cfg)
A = ctx.new_matrix()
plan = ctx.default_plan()
cnt = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64, device=ctx.device)
ctx.run(A, plan=plan, counters=cnt)
torch.cuda.synchronize()
print(name, "events", int(cnt[0]))
