"""Device time of each streaming layer range of assemble() (R4 default),
and of each colour group inside it.

    python tools/range_timing.py [R4] [fracs]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2101_08825_b200 import _native as N  # noqa: E402
from paper_2101_08825_b200.assembly import AssemblyContext  # noqa: E402
from paper_2101_08825_b200.device import ColorPlan  # noqa: E402
from paper_2101_08825_b200.parallel import (pair_counts,  # noqa: E402
                                            slab_layers_fracs)

name = sys.argv[1] if len(sys.argv) > 1 else "R4"
fracs = [float(x) for x in (sys.argv[2] if len(sys.argv) > 2 else
                            "0.5,0.8,0.93,1.0").split(",")]
mesh, space, kp, cfg = bench.build_problem(name)
dev = torch.device("cuda", 0)
ctx = AssemblyContext(mesh, space, kp, cfg, dev)
A = ctx.new_matrix()
work = pair_counts(mesh, kp, ctx.dmesh)
layers = slab_layers_fracs(mesh, fracs, None)
plan = ColorPlan(mesh, None, dev, work=work, layers=layers)
cnt = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64, device=dev)
print("layers", layers)
for trial in range(2):
    A._dvals.zero_()
    evs = []
    for s, _ in enumerate(layers):
        g0, g1 = plan.group_range(s)
        for g in range(g0, g1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.run(A, plan=plan, counters=cnt, groups=(g, g + 1))
            e1.record()
            evs.append((s, g, e0, e1))
    torch.cuda.synchronize()
    per = {}
    for s, g, e0, e1 in evs:
        per.setdefault(s, []).append(e0.elapsed_time(e1))
    for s in sorted(per):
        ms = per[s]
        n = int(plan.color_ptr[(s + 1) * plan.NCOLORS] -
                plan.color_ptr[s * plan.NCOLORS])
        print(f"trial {trial} range {s} {layers[s]}: {sum(ms):8.1f} ms, "
              f"{n} elements, groups min/max {min(ms):.1f}/{max(ms):.1f} ms",
              flush=True)
