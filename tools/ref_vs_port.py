"""Per-thread speed of the oracle port vs the live reference (numba).

Runs in the build container only (needs /root/reference or baseline/_ref).
Same seeded outer sample of a workload, one thread each:
  reference  mollifem.assembly._run_general (numba _general_core)
  port       oracle/mf_oracle.c orc_general_core
and checks the two value arrays are bit-identical.

    python tools/ref_vs_port.py [--config R4-small] [--n 60] [--reps 3]
"""

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="R4-small")
    ap.add_argument("--n", type=int, default=60)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import bench
    import oracle
    from bench import ref_import
    mf = ref_import()
    from mollifem import assembly as RA
    mesh, space, kp, cfg = bench.build_problem(args.config)
    rmesh, rspace, rkp, rcfg = bench.build_reference_problem(mf, args.config)
    rng = np.random.default_rng(0)
    outer = np.sort(rng.choice(rmesh.n_elements, args.n, replace=False))
    prep = RA._Prep(rmesh, rspace, rkp, rcfg)
    # JIT warm-up on the same arrays (a few elements)
    A0 = RA._new_matrix(rmesh, rspace, rkp, rcfg)
    RA._run_general(rmesh, rspace, rkp, rcfg, prep, A0, outer_ids=outer[:2])
    ptr, _ = oracle.candidates(mesh, kp.delta + kp.eps, outer,
                               np.ones(mesh.n_elements, np.uint8))
    pairs = int(ptr[-1])
    t_ref, t_port = [], []
    for _ in range(args.reps):
        A = RA._new_matrix(rmesh, rspace, rkp, rcfg)
        t = time.perf_counter()
        ev_r = RA._run_general(rmesh, rspace, rkp, rcfg, prep, A,
                               outer_ids=outer)
        t_ref.append(time.perf_counter() - t)
        from paper_2101_08825_b200.assembly import HostPattern
        B = HostPattern.for_space(mesh, space, kp, cfg)
        t = time.perf_counter()
        ev_p = oracle.run_general(mesh, space, kp, cfg, B, outer_ids=outer)
        t_port.append(time.perf_counter() - t)
    same = bool(np.array_equal(A.vals, B.vals)) and ev_r == ev_p
    r, p = min(t_ref), min(t_port)
    print(f"{args.config}: {args.n} outer elements, {pairs} pairs, "
          f"{ev_r} events; bit-identical: {same}")
    print(f"  reference numba : {r:.3f} s  {pairs / r:.4g} pairs/s/thread")
    print(f"  oracle port     : {p:.3f} s  {pairs / p:.4g} pairs/s/thread  "
          f"(port/ref speed {r / p:.3f})")


if __name__ == "__main__":
    main()
