"""A/B timing of library variants on one workload (GPU box).

    python tools/ab_time.py --config R4-half --reps 3 lib1.so lib2.so ...

Each variant runs in its own process (MF_LIB_PATH selects the .so); the
device time of one full assembly (ctx.run over all colours, CUDA events),
the event count and a value checksum are printed, plus the relative
Frobenius distance of each variant's values to the first variant's."""

import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg, reps, out):
    sys.path.insert(0, ROOT)
    import torch
    import bench
    from paper_2101_08825_b200 import _native as N
    from paper_2101_08825_b200.assembly import AssemblyContext
    mesh, space, kp, c = bench.build_problem(cfg)
    ctx = AssemblyContext(mesh, space, kp, c)
    A = ctx.new_matrix()
    plan = ctx.default_plan()
    cnt = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64, device=ctx.device)
    ts = []
    for r in range(reps + 1):
        A._dvals.zero_()
        cnt.zero_()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        ctx.run(A, plan=plan, counters=cnt)
        e.record()
        e.synchronize()
        if r:
            ts.append(s.elapsed_time(e))
    v = A._dvals
    np.save(out, v.cpu().numpy())
    print(json.dumps({"ms": ts, "events": int(cnt[0]),
                      "counters": cnt.cpu().tolist(),
                      "norm": float(torch.linalg.vector_norm(v))}))


def main():
    if sys.argv[1] == "--child":
        return child(sys.argv[2], int(sys.argv[3]), sys.argv[4])
    args = sys.argv[1:]
    cfg, reps = "R4-half", 3
    if args[0] == "--config":
        cfg, args = args[1], args[2:]
    if args[0] == "--reps":
        reps, args = int(args[1]), args[2:]
    base = None
    for i, lib in enumerate(args):
        out = f"/tmp/ab_{i}.npy"
        env = dict(os.environ, MF_LIB_PATH=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child", cfg,
                            str(reps), out], env=env, capture_output=True,
                           text=True)
        if r.returncode:
            print(lib, "FAILED", r.stderr[-1500:])
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        v = np.load(out)
        os.remove(out)   # R4-tet values are 16 GB per variant
        if base is None:
            base = v
        rel = float(np.linalg.norm(v - base) / np.linalg.norm(base))
        print(f"{lib}: ms {min(d['ms']):.1f} (all {[round(x, 1) for x in d['ms']]})"
              f" events {d['events']} relF-vs-first {rel:.2e} "
              f"counters {d['counters']}", flush=True)


if __name__ == "__main__":
    main()
