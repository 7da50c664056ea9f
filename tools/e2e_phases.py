"""Time assemble() end to end for the two strategies (diagnostic)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2101_08825_b200 import assemble, AssemblyConfig
name = sys.argv[1] if len(sys.argv) > 1 else "R4"
strats = sys.argv[2].split(",") if len(sys.argv) > 2 else ["blocked"]
mesh, space, kp, cfg = bench.build_problem(name)
dev = torch.device("cuda", 0)
def T(): torch.cuda.synchronize(); return time.perf_counter()
for strat in strats:
    c = AssemblyConfig(L_max=cfg.L_max, outer_rule=cfg.outer_rule, inner_rule=cfg.inner_rule, strategy=strat)
    for trial in range(3):
        t = T(); B = assemble(mesh, space, kp, c, device=dev); t3 = T()
        print(f"{name} assemble {strat} trial {trial}: {t3-t:.3f}s  vals[123]={B.vals[123]:.6e} events={B.events}", flush=True)
        del B
