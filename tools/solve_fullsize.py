"""Time the manufactured-solution pipeline at full size on the device:
assemble -> assemble_rhs -> solve -> L2 error (u = |x|^2, f = -2 kappa dim).

    python tools/solve_fullsize.py [R4]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2101_08825_b200 import assemble, assemble_rhs, solve  # noqa: E402
from paper_2101_08825_b200.fe_space import l2_error  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "R4"
mesh, space, kp, cfg = bench.build_problem(name)
dim, kappa = mesh.dim, kp.kappa


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


f = lambda x: np.full(x.shape[:-1], -2.0 * kappa * dim)
u_ex = lambda x: (x ** 2).sum(axis=-1)
t0 = T()
A = assemble(mesh, space, kp, cfg, keep_on_device=True)
t1 = T()
rhs = assemble_rhs(mesh, space, kp, f, u_ex, A)
t2 = T()
u, rep = solve(A, rhs, space.free, space.constrained,
               u_ex(space.dof_coords[space.constrained]))
t3 = T()
err = l2_error(space, u, u_ex)
print(f"{name}: assemble {t1 - t0:.2f}s rhs {t2 - t1:.2f}s solve "
      f"{t3 - t2:.2f}s ({rep}) L2 error {err:.3e}", flush=True)
