"""Benchmark: interacting element pairs/s of the nonlocal stiffness assembly.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config R4]
                    [--impl ours|reference]

Metric (BASELINE.json): interacting element-pairs/sec and full assembly
time, FP64 roofline fraction.  A *pair* is one (outer l, inner m) entry of
the reference candidate lists (`_candidates`, assembly.py:157-175), the
numerator for both the GPU and the CPU; a *step* is one full assembly of
A = 2(A21 + A22) for the workload.

  value  inputs resident in HBM: zero vals, mf_general_core over all
         colours (neighbour search fused), asymmetry diagnostic.
  e2e    the public API `assemble(mesh, space, kernel, config)` from host
         arrays to a populated host SparseMatrix: mesh/DOF upload, the
         same kernels, D2H of the 8-byte values.

Default workload R4 = BASELINE config #4 stand-in (3D hex Q1, 64^3 cells,
delta=0.1, eps=h/2, kappa=2, GL3, L_max=2).  Multi-GPU:
inner elements are split into z-slabs balanced by pair count, one per rank;
each rank assembles the rows its slab touches; the timed step includes the
one interface-plane send/recv per slab boundary (parallel.py).  e2e at N>1
is `assemble_distributed` (upload, slab assembly, exchange, NCCL row-block
gather to rank 0, D2H on rank 0).

The CPU leg (cpu_baseline / --impl reference) times the UNMODIFIED
reference (numba, installed under baseline/_ref) on a seeded sample of
outer elements with all host threads -- its general path, the comparison
path of the GPU design -- and, once, its default assemble() (strategy
"auto" -> offset-blocked) in full on a smaller workload
(cpu_baseline.default_path).  Workloads the reference cannot build (tets,
Delaunay) fall back to the oracle port (oracle/mf_oracle.c, within 10-20%
of numba per thread, tools/ref_vs_port.py).  On structured meshes the GPU
line also reports e2e_default_path: our assemble(strategy="auto").
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (dim, omega, h, delta, eps, kappa, kind, L_max, rule)
    "R1": (2, ((0.0, 1.0),) * 2, 1 / 32, 0.1, 1 / 64, 1.0, "tri", 3,
           "default"),
    # BASELINE config #1 as written: the 3-point triangle rule ("tri3";
    # the reference maps every triangle preset to Dunavant-7)
    "R1-tri3": (2, ((0.0, 1.0),) * 2, 1 / 32, 0.1, 1 / 64, 1.0, "tri", 3,
                "tri3"),
    "R3-2h": (2, ((0.0, 1.0),) * 2, 1 / 512, 2 / 512, 1 / 1024, 1.0, "tri",
              3, "default"),
    "R3-4h": (2, ((0.0, 1.0),) * 2, 1 / 512, 4 / 512, 1 / 1024, 1.0, "tri",
              3, "default"),
    "R3-8h": (2, ((0.0, 1.0),) * 2, 1 / 512, 8 / 512, 1 / 1024, 1.0, "tri",
              3, "default"),
    "R3-16h": (2, ((0.0, 1.0),) * 2, 1 / 512, 16 / 512, 1 / 1024, 1.0, "tri",
               3, "default"),
    "R4": (3, ((0.0, 1.0),) * 3, 1 / 64, 0.1, 1 / 128, 2.0, "hex", 2,
           "default"),
    "R4-gauss2": (3, ((0.0, 1.0),) * 3, 1 / 64, 0.1, 1 / 128, 2.0, "hex", 2,
                  "gauss2"),
    "R4-small": (3, ((0.0, 0.25),) * 3, 1 / 64, 0.1, 1 / 128, 2.0, "hex", 2,
                 "default"),
    # Omega = [0, 0.5]^3 (46^3 hexes): kernel A/B timing stand-in for R4
    "R4-half": (3, ((0.0, 0.5),) * 3, 1 / 64, 0.1, 1 / 128, 2.0, "hex", 2,
                "default"),
    "R5": (3, ((0.0, 1.0),) * 3, 1 / 128, 4 / 128, 1 / 512, 2.0, "hex", 2,
           "default"),
    # BASELINE config #4 as written: 6-tet P1 cubes, 4-point tet rule
    "R4-tet": (3, ((0.0, 1.0),) * 3, 1 / 64, 0.1, 1 / 128, 2.0, "tet", 2,
               "tet4"),
    "R4-tet-small": (3, ((0.0, 0.25),) * 3, 1 / 64, 0.1, 1 / 128, 2.0,
                     "tet", 2, "tet4"),
    # BASELINE config #5 (jittered tets, delta = 4h, eps = h/4, 11-point
    # rule) at half its resolution (64^3 cubes instead of 128^3; the full
    # size is ~1.3e11 pairs and a 47 GB matrix)
    "R5-tet-64": (3, ((0.0, 1.0),) * 3, 1 / 64, 4 / 64, 1 / 256, 2.0, "tet",
                  2, "tet11"),
    "R5-tet-small": (3, ((0.0, 0.25),) * 3, 1 / 64, 4 / 64, 1 / 256, 2.0,
                     "tet", 2, "tet11"),
    # BASELINE config #5 at full size on one GPU: 128^3 cubes (+5 Gamma
    # rings) x 6 tets = 15.8M tets, ~1.3e11 pairs, 47 GB matrix
    "R5-tet": (3, ((0.0, 1.0),) * 3, 1 / 128, 4 / 128, 1 / 512, 2.0, "tet",
               2, "tet11"),
    # BASELINE config #2: unstructured Delaunay P1 mesh of ~200k seeded
    # jittered points (400^2 Omega lattice + 21 Gamma rings = 442^2 =
    # 195,364 vertices), delta = 0.05, eps = h/2, 6-point rule, L_max 3
    "R2": (2, ((0.0, 1.0),) * 2, 1 / 400, 0.05, 1 / 800, 1.0, "delaunay",
           3, "tri6"),
    "R2-small": (2, ((0.0, 0.25),) * 2, 1 / 400, 0.05, 1 / 800, 1.0,
                 "delaunay", 3, "tri6"),
}
# vertex jitter (fraction of h, seeded) per workload (tet meshes only)
JITTER = {"R5-tet-64": 0.1, "R5-tet-small": 0.1, "R5-tet": 0.1, "R2": 0.3,
          "R2-small": 0.3}

METRIC = "interacting element-pairs/sec (full nonlocal stiffness assembly)"

# total candidate pairs per workload (GPU counters; R1/R4-small are
# re-checked against the oracle's _candidates count in tests/test_bench.py)
PAIRS = {"R1": 462400, "R3-2h": 52243984, "R3-4h": 130507776,
         "R3-8h": 398401600, "R3-16h": 1414361664, "R4": 1382469544,
         "R4-gauss2": 1382469544, "R4-small": 61162984, "R5": None}


def build_problem(name):
    from paper_2101_08825_b200 import (AssemblyConfig, FESpace, KernelParams,
                                       build_mesh)
    dim, om, h, delta, eps, kappa, kind, lmax, rule = CONFIGS[name]
    kp = KernelParams(dim, delta, eps, kappa)
    if kind == "delaunay":
        from paper_2101_08825_b200.mesh import build_delaunay_mesh
        mesh = build_delaunay_mesh(om, h, delta + eps, jitter=JITTER[name],
                                   seed=0)
    else:
        mesh = build_mesh(dim, om, h, delta + eps, kind,
                          jitter=JITTER.get(name, 0.0), seed=0)
    space = FESpace(mesh, 1)
    cfg = AssemblyConfig(L_max=lmax, outer_rule=rule, inner_rule=rule,
                         strategy="general")
    return mesh, space, kp, cfg


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def ref_import():
    """The unmodified reference package (numba) installed under
    baseline/_ref; None if it is not installed."""
    os.environ.setdefault("NUMBA_CACHE_DIR",
                          os.path.join("/tmp", "mf_numba_cache"))
    extra = [REF_DIR] + [p for p in (os.environ.get("MF_REF_PATH"),) if p]
    for p in extra:
        if os.path.isdir(os.path.join(p, "mollifem")) and p not in sys.path:
            sys.path.insert(0, p)
    try:
        import mollifem
        import numba  # noqa: F401
    except ImportError:
        return None
    return mollifem


def build_reference_problem(mf, name):
    """The workload built by the reference's own host layer (structured
    quad/tri/hex meshes only; None for tets and Delaunay meshes, which the
    reference cannot build)."""
    dim, om, h, delta, eps, kappa, kind, lmax, rule = CONFIGS[name]
    if kind not in ("tri", "quad", "hex") or name in JITTER or \
            rule in ("tri3", "tri6"):
        return None
    mesh = mf.build_mesh(dim, om, h, delta + eps, kind)
    space = mf.FESpace(mesh, 1)
    kp = mf.KernelParams(dim, delta, eps, kappa)
    cfg = mf.AssemblyConfig(L_max=lmax, outer_rule=rule, inner_rule=rule,
                            strategy="general")
    return mesh, space, kp, cfg


def config_json(name, mesh, space, n_gpus, slab_info=None,
                strategy="general"):
    dim, om, h, delta, eps, kappa, kind, lmax, rule = CONFIGS[name]
    mdesc = f"{kind} structured"
    if kind == "delaunay":
        mdesc = (f"unstructured Delaunay P1 triangles of "
                 f"{len(mesh.nodes)} seeded lattice points jittered "
                 f"+-{JITTER[name]}h (seed 0)")
    if kind == "tet":
        mdesc = "6-tet (Kuhn) cubes" + (
            f", vertices jittered +-{JITTER[name]}h (seed 0)"
            if name in JITTER else "")
    d = {"workload": name, "strategy": strategy, "dim": dim, "mesh": mdesc,
         "cells": list(mesh.grid_ncells), "elements": mesh.n_elements,
         "n_dofs": space.n_dofs, "fe_degree": 1, "h": h, "delta": delta,
         "eps": eps, "kappa": kappa, "L_max": lmax,
         "rule": ({"tri3": "strang3", "tri6": "dunavant6"}.get(rule,
                                                               "dunavant7")
                  if kind in ("tri", "delaunay") else rule),
         "parallelism": f"z-slab x{n_gpus}" if n_gpus > 1 else "single",
         "l2": "value array > L2 (rewritten every step)"}
    if slab_info:
        d.update(slab_info)
    return d


# --------------------------------------------------------------------------
# clocks sampling during the timed region

class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,"
         "clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": mx, "samples": len(sm),
                "reasons": sorted(reasons)}


# --------------------------------------------------------------------------
# flop model: executed arithmetic of the kernels

def flop_model(name, counters):
    """(executed_flops, canonical_flops) for one assembly.

    canonical = SURVEY.md 8(d) (reference rank-1 form, every event);
    executed  = what mf_hex.cu / mf_2d.cu actually issue per event class
    (sum-factorised full events, rank-1 plateau events, dead events 0),
    counting mul/add/sub as 1 and FMA as 2, sqrt/div/shell polynomial
    not counted (same convention as the canonical count)."""
    from paper_2101_08825_b200 import _native as N
    dim = CONFIGS[name][0]
    ev = int(counters[N.CNT_EVENTS])
    pairs = int(counters[N.CNT_PAIRS])
    full = int(counters[N.CNT_EV_FULL])
    plat = int(counters[N.CNT_EV_PLATEAU]) + int(counters[N.CNT_EV_UPPER])
    rule = CONFIGS[name][8]
    if CONFIGS[name][6] == "tet":
        nq = {"tet1": 1, "tet4": 4, "tet11": 11}[rule]
        nq1 = nq2 = nq
        nl = 4
        canon_ev = nq2 * nq1 * (3 * dim - 1 + 3) + 2 * nq2 * nq1 * nl \
            + 2 * nq2 * nl * nl
        canon_pair = 2 * nq1 * nl * nl
        # per point pair: 3 sub, 3 mul, 2 add, 4 FMA; per q2: ~40 (map,
        # pullback, weights)
        f_full = nq2 * (nq1 * (8 + 8) + 40)
        f_plat = nq2 * 40
        f_pair = 2 * nl * nl * nq1 + nq1 * nl + 60
    elif dim == 3:
        no = ni = 2 if rule == "gauss2" else 3
        nq1, nq2, nl = ni ** 3, no ** 3, 8
        canon_ev = nq2 * nq1 * (3 * dim - 1 + 3) + 2 * nq2 * nq1 * nl \
            + 2 * nq2 * nl * nl
        canon_pair = 2 * nq1 * nl * nl
        # per lane: sq (2*3NO), sxy (NO^2), d2 (NO^3), x-contraction
        # (2 FMA per point), y (4*NO FMA per c), z (8 FMA per c)
        lane = 6 * no + no * no + no ** 3 + 4 * no ** 3 + 8 * no * no \
            + 16 * no
        f_full = nq1 * lane + 3 * no * 8
        f_plat = 3 * no * 8 + 6 * no + 16
        f_pair = 2 * 2 * nq1 * 64 + 8 * nq1
    else:
        nq1 = nq2 = {"tri6": 6, "tri3": 3}.get(rule, 7)
        nl = 3
        canon_ev = nq2 * nq1 * (3 * dim - 1 + 3) + 2 * nq2 * nq1 * nl \
            + 2 * nq2 * nl * nl
        canon_pair = 2 * nq1 * nl * nl
        # per point pair: 2 sub, 2 mul, 1 add, 3 FMA; per q2: ~14
        f_full = nq2 * (nq1 * (5 + 6) + 14)
        f_plat = nq2 * 16
        f_pair = 2 * nl * nl * nq1 + nq1 * nl
    executed = full * f_full + plat * f_plat + pairs * f_pair
    canonical = ev * canon_ev + pairs * canon_pair
    return executed, canonical


def canonical_event_flops(name):
    """SURVEY.md 8(d) F_event of one event of this workload."""
    dim, kind, rule = CONFIGS[name][0], CONFIGS[name][6], CONFIGS[name][8]
    if kind == "tet":
        nq1 = nq2 = {"tet1": 1, "tet4": 4, "tet11": 11}[rule]
        nl = 4
    elif dim == 3:
        nq1 = nq2 = (2 if rule == "gauss2" else 3) ** 3
        nl = 8
    else:
        nq1 = nq2 = {"tri6": 6, "tri3": 3}.get(rule, 7)
        nl = 3
    return nq2 * nq1 * (3 * dim - 1 + 3) + 2 * nq2 * nq1 * nl \
        + 2 * nq2 * nl * nl


def fp64_peak(device):
    """Measured sustained DFMA rate (TF/s) with mf_fp64_probe."""
    import torch
    from paper_2101_08825_b200 import _native as N
    L = N.lib()
    out = torch.zeros(1, dtype=torch.float64, device=device)
    blocks, threads, iters = 148 * 8, 256, 40000
    st = N.stream_ptr()
    N.check(L.mf_fp64_probe(N.ptr(out), iters, blocks, threads, st), "probe")
    best = 0.0
    for _ in range(3):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        N.check(L.mf_fp64_probe(N.ptr(out), iters, blocks, threads, st),
                "probe")
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e)
        best = max(best, L.mf_fp64_probe_flops(iters, blocks, threads) /
                   (ms * 1e-3) / 1e12)
    return best


# --------------------------------------------------------------------------
# CPU leg (oracle port on the host cores)

def cpu_sample(name, mesh, space, kp, cfg, budget_s=20.0, seed=0,
               use_reference=True):
    """cpu_baseline of the GPU line: the unmodified reference (numba) on a
    seeded sample when it is installed and can build the workload, else
    the oracle port (oracle/mf_oracle.c)."""
    if use_reference:
        mf = ref_import()
        if mf is not None and build_reference_problem(mf, name) is not None:
            return RefRunner(mf, name).sample(budget_s, seed)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    from paper_2101_08825_b200.assembly import HostPattern
    oracle.build()
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    n = mesh.n_elements
    A = HostPattern.for_space(mesh, space, kp, cfg)
    private = A.nnz * 8 * threads < 8e9
    # calibrate on a small sample, then size the timed one to the budget
    probe = np.sort(rng.choice(n, min(n, 4 * threads), replace=False))
    p_ptr, _ = oracle.candidates(mesh, kp.delta + kp.eps, probe,
                                 np.ones(n, np.uint8))
    _, dt = oracle.run_general_threads(mesh, space, kp, cfg, A, probe,
                                       threads, private=False, blk=1)
    rate = max(p_ptr[-1] / max(dt, 1e-6), 1.0)
    want_pairs = rate * budget_s
    per_el = max(p_ptr[-1] / len(probe), 1.0)
    k = int(min(n, max(threads, want_pairs / per_el)))
    sample = np.sort(rng.choice(n, k, replace=False))
    ptr, _ = oracle.candidates(mesh, kp.delta + kp.eps, sample,
                               np.ones(n, np.uint8))
    A.vals[:] = 0.0
    ev, dt = oracle.run_general_threads(mesh, space, kp, cfg, A, sample,
                                        threads, private=private, blk=1)
    pairs = int(ptr[-1])
    return {"value": pairs / dt, "unit": "pairs/s", "cores": threads,
            "kind": "port", "seconds": dt,
            "sample": (f"{k} seeded outer elements (rng 0) of {name} "
                       f"= {pairs} pairs, {ev} events, "
                       f"{'private' if private else 'shared'} value "
                       "buffers, oracle/mf_oracle.c (C restatement of "
                       "_general_core, no FMA) on all host threads")}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


class RefRunner:
    """The unmodified reference (numba, baseline/_ref) on the host cores.

    General path (the per-pair comparison path of the GPU design, SURVEY
    8(d) CPU plan item 3): a seeded sample of outer elements split over
    all host threads, each thread calling the reference's own
    `_run_general(outer_ids=...)` (assembly.py:369-388; nogil numba
    `_candidates` + `_general_core`), as `parallel_assemble` does with its
    thread pool (parallel.py:157-178).  Default path (item 2): the
    reference `assemble()` with strategy "auto" -> offset-blocked
    (assembly.py:448-473), timed in full on a workload small enough to
    finish in seconds and reported as pairs/s."""

    def __init__(self, mf, name):
        from mollifem import assembly as RA
        self.mf, self.RA, self.name = mf, RA, name
        t = time.perf_counter()
        self.mesh, self.space, self.kp, self.cfg = build_reference_problem(
            mf, name)
        self.prep = RA._Prep(self.mesh, self.space, self.kp, self.cfg)
        # one shared value buffer (the sampled rows are a timing workload;
        # R4's 16.4 GB pattern cannot be replicated per thread)
        self.A = RA._new_matrix(self.mesh, self.space, self.kp, self.cfg)
        self.setup_s = time.perf_counter() - t
        self.threads = os.cpu_count() or 1
        n = self.mesh.n_elements
        # JIT warm-up (numba compiles per signature on first call)
        RA._run_general(self.mesh, self.space, self.kp, self.cfg, self.prep,
                        self.A, outer_ids=np.arange(min(2, n)))
        probe = np.random.default_rng(12345).choice(
            n, min(n, 6 * self.threads), replace=False)
        self.rate = None
        pairs, dt, _ = self._run(np.sort(probe))
        self.rate = pairs / max(dt, 1e-6)
        self.per_el = max(pairs / len(probe), 1.0)

    def _run(self, sample):
        from concurrent.futures import ThreadPoolExecutor
        RA = self.RA
        reach = self.kp.delta + self.kp.eps
        mask = np.ones(self.mesh.n_elements, dtype=np.bool_)
        ptr, _ = RA._candidates(self.mesh, reach, sample, mask)
        chunks = [c for c in np.array_split(sample, self.threads) if c.size]

        def work(c):
            return RA._run_general(self.mesh, self.space, self.kp, self.cfg,
                                   self.prep, self.A, outer_ids=c)

        with ThreadPoolExecutor(max_workers=len(chunks)) as pool:
            t = time.perf_counter()
            ev = sum(pool.map(work, chunks))
            dt = time.perf_counter() - t
        return int(ptr[-1]), dt, int(ev)

    def sample(self, budget_s, seed):
        n = self.mesh.n_elements
        k = int(min(n, max(self.threads, self.rate * budget_s / self.per_el)))
        rng = np.random.default_rng(seed)
        s = np.sort(rng.choice(n, k, replace=False))
        pairs, dt, ev = self._run(s)
        return {"value": pairs / dt, "unit": "pairs/s",
                "cores": self.threads, "kind": "reference",
                "cpu_model": cpu_model(), "seconds": dt,
                "sample": (f"{k} seeded outer elements (rng {seed}) of "
                           f"{self.name} = {pairs} pairs, {ev} events; "
                           "unmodified reference mollifem "
                           "_run_general (numba _general_core, nogil) on "
                           f"{len(np.array_split(s, self.threads))} host "
                           "threads, one shared value buffer")}

    def default_path(self, name="R4-small"):
        """Reference default assemble() (strategy auto -> blocked) timed in
        full on `name` (JIT warmed on the same mesh first)."""
        mf = self.mf
        rp = build_reference_problem(mf, name)
        if rp is None:
            return None
        mesh, space, kp, cfg = rp
        auto = mf.AssemblyConfig(L_max=cfg.L_max, outer_rule=cfg.outer_rule,
                                 inner_rule=cfg.inner_rule, strategy="auto")
        small = build_reference_problem(mf, "R1") if mesh.dim == 2 else None
        if small is not None:
            mf.assemble(small[0], small[1], small[2], auto)
        else:
            # warm the blocked JIT on a tiny mesh of the same dim and kind
            dim, om, h, delta, eps, kappa, kind, lmax, rule = CONFIGS[name]
            tiny = mf.build_mesh(dim, ((0.0, 4 * h),) * dim, h,
                                 delta + eps, kind)
            mf.assemble(tiny, mf.FESpace(tiny, 1), kp, auto)
        reach = kp.delta + kp.eps
        ptr, _ = self.RA._candidates(
            mesh, reach, np.arange(mesh.n_elements),
            np.ones(mesh.n_elements, dtype=np.bool_))
        t = time.perf_counter()
        A = mf.assemble(mesh, space, kp, auto)
        dt = time.perf_counter() - t
        pairs = int(ptr[-1])
        return {"value": pairs / dt, "unit": "pairs/s", "cores": 1,
                "workload": name, "pairs": pairs, "seconds": dt,
                "events": int(A.events),
                "path": "reference default assemble(strategy='auto') -> "
                        "offset-blocked (_run_blocked), single thread, "
                        "full assembly incl. _finish"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.config
    mf = ref_import()
    if mf is None or build_reference_problem(mf, name) is None:
        return run_reference_port(args)
    runner = RefRunner(mf, name)
    vals = []
    for i in range(args.warmup + args.steps):
        r = runner.sample(args.ref_step_budget if i >= args.warmup else 1.0,
                          seed=i)
        if i >= args.warmup:
            vals.append(r)
    v = statistics.median(x["value"] for x in vals)
    total_pairs = PAIRS.get(name) or v
    dflt = None
    if not args.no_default_path:
        dname = DEFAULT_PATH_WORKLOAD.get(name, name)
        dflt = runner.default_path(dname)
        if dflt is not None and total_pairs:
            dflt["projected_seconds_full_workload"] = total_pairs / dflt[
                "value"]
    cb = dict(vals[0])
    cb["value"] = v
    if dflt is not None:
        cb["default_path"] = dflt
    line = {"metric": METRIC, "value": v, "unit": "pairs/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.median(x["seconds"] for x in vals) * 1e3,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": config_json(name, runner.mesh, runner.space, 1),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "projected_full_assembly_s": (total_pairs / v
                                          if PAIRS.get(name) else None),
            "note": ("each step = the reference general path on a bounded "
                     "seeded sample of outer elements (ms_per_step is that "
                     "sample's wall time); projected_full_assembly_s = all "
                     "pairs at the sampled rate")}
    print(json.dumps(line), flush=True)


# workload on which the reference default (blocked) path is timed in full
DEFAULT_PATH_WORKLOAD = {"R4": "R4-small", "R4-gauss2": "R4-small",
                         "R5": "R4-small", "R3-16h": "R3-2h",
                         "R3-8h": "R3-2h", "R3-4h": "R3-2h"}


def run_reference_port(args):
    """Fallback when the reference cannot run here (not installed, or a
    workload it cannot build: tets, Delaunay): the oracle port."""
    name = args.config
    mesh, space, kp, cfg = build_problem(name)
    total_pairs = PAIRS.get(name)
    if total_pairs is None:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle
        n = mesh.n_elements
        ptr, _ = oracle.candidates(mesh, kp.delta + kp.eps, np.arange(n),
                                   np.ones(n, np.uint8))
        total_pairs = int(ptr[-1])
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(name, mesh, space, kp, cfg,
                       budget_s=(args.ref_step_budget if i >= args.warmup
                                 else 1.0),
                       seed=i, use_reference=False)
        if i >= args.warmup:
            vals.append(r)
    v = statistics.median(x["value"] for x in vals)
    cb = dict(vals[0])
    cb["value"] = v
    line = {"metric": METRIC, "value": v, "unit": "pairs/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.median(x["seconds"] for x in vals) * 1e3,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": config_json(name, mesh, space, 1),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "projected_full_assembly_s": total_pairs / v,
            "note": ("the reference cannot build this workload (or is not "
                     "installed): oracle port on a seeded sample")}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# GPU leg

def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2101_08825_b200 import _native as N
    from paper_2101_08825_b200 import assemble
    from paper_2101_08825_b200.assembly import AssemblyContext
    from paper_2101_08825_b200.device import ColorPlan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    name = args.config
    mesh, space, kp, cfg = build_problem(name)
    stream = torch.cuda.current_stream()
    slab = None
    if world == 1:
        ctx = AssemblyContext(mesh, space, kp, cfg, dev)
        A = ctx.new_matrix()
        plan = ctx.default_plan()
        counters = torch.zeros(N.MF_NCOUNTERS, dtype=torch.int64, device=dev)
        n_launch = (np.count_nonzero(np.diff(plan.color_ptr))
                    * launches_per_group(mesh)) + 1
        if args.strategy == "blocked":
            n_launch = 2 + np.count_nonzero(np.diff(plan.color_ptr))

        def work():
            A._dvals.zero_()
            counters.zero_()
            if args.strategy == "blocked":
                ctx.run_blocked(A, counters=counters)
            else:
                ctx.run(A, plan=plan, counters=counters)

        def finish():
            ctx.finish(A, counters)
            return A.counters
    else:
        from paper_2101_08825_b200.device import DeviceMesh
        from paper_2101_08825_b200.parallel import SlabAssembler, pair_counts
        w = pair_counts(mesh, kp, DeviceMesh(mesh, space, dev))
        sa = SlabAssembler(mesh, space, kp, cfg, rank, world, dev, weights=w)
        ctx = sa.ctx
        plan = sa.color_plan
        slab = {"slab_layers": [list(x) for x in sa.layers],
                "interface_plane_bytes": int(
                    (sa.plan.send_range[1] - sa.plan.send_range[0]) * 8
                    if sa.plan.send_range else 0)}
        n_launch = (np.count_nonzero(np.diff(plan.color_ptr))
                    * launches_per_group(mesh))

        def work():
            sa.assemble_local()
            sa.exchange()

        def finish():
            return sa.counters.cpu().numpy()

    def step():
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        work()
        e.record(stream)
        cnt = finish()
        return s, e, cnt

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        evs = [step() for _ in range(args.steps)]
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1) / args.steps
    kern_ms = [s.elapsed_time(e) for s, e, _ in evs]
    cnt = evs[-1][2]
    pairs = int(cnt[N.CNT_PAIRS])
    if world > 1:
        t = torch.tensor([ms, float(pairs)], dtype=torch.float64, device=dev)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_all, pairs_all = float(mx[0]), int(sm[1])
    else:
        ms_all, pairs_all = ms, pairs
    value = pairs_all / (ms_all * 1e-3)

    # ---- end to end through the public API (host in, host out) --------
    e2e = None
    if not args.no_e2e:
        from paper_2101_08825_b200.parallel import assemble_distributed

        def api_call():
            if world == 1:
                c = cfg
                if args.strategy == "blocked":
                    from paper_2101_08825_b200 import AssemblyConfig
                    c = AssemblyConfig(L_max=cfg.L_max,
                                       outer_rule=cfg.outer_rule,
                                       inner_rule=cfg.inner_rule,
                                       strategy="blocked")
                return assemble(mesh, space, kp, c, device=dev)
            return assemble_distributed(mesh, space, kp, cfg)

        B = api_call()
        del B
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        t = time.perf_counter()
        for _ in range(e2e_steps):
            B = api_call()
            if B is not None:
                _ = B.vals[-1]
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t) / e2e_steps
        if world > 1:
            tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt[0])
        from paper_2101_08825_b200.device import DeviceMesh
        h2d = (ctx.h2d_bytes + plan.h2d_bytes) * world
        nnz = int(np.asarray(ctx_nnz(mesh, space, kp, cfg)))
        e2e = {"value": pairs_all / e2e_s, "unit": "pairs/s",
               "seconds_per_assembly": e2e_s,
               "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(nnz * 8 + 8 * N.MF_NCOUNTERS)}
        del B

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak = fp64_peak(dev)
    executed, canonical = flop_model(name, cnt)
    kms = statistics.mean(kern_ms)
    achieved = executed / (kms * 1e-3) / 1e12
    prof = load_traffic(name)
    if args.strategy == "blocked":
        # scatter-bound: algorithmic bytes = one read+write of every value
        nnz = ctx_nnz(mesh, space, kp, cfg)
        roof = {"bound": "hbm", "achieved": 16.0 * nnz / (kms * 1e-3) / 1e9,
                "peak": hbm_peak(), "unit": "GB/s", "traffic": None,
                "kernel_ms": kms,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (or fallback)"}
        roof["frac"] = roof["achieved"] / roof["peak"]
    else:
        # achieved = SURVEY.md 8(d)'s canonical per-event / per-pair flop
        # figure x this launch's events and pairs (the algorithmic count);
        # executed_* is what the kernels actually issue after sum
        # factorisation and the dead/plateau proofs
        canon_tf = canonical / (kms * 1e-3) / 1e12
        # the canonical count credits every event with the reference's
        # rank-1 point-pair arithmetic, including the dead events (gap >=
        # delta+eps at every point pair) on which the reference itself does
        # no arithmetic (_kernels.py:134-135); the live count leaves them out
        live = canonical - int(cnt[N.CNT_EV_DEAD]) * canonical_event_flops(
            name)
        roof = {"bound": "fp64", "achieved": canon_tf, "peak": peak,
                "unit": "TFLOP/s", "frac": canon_tf / peak,
                "live_canonical_tflops": live / (kms * 1e-3) / 1e12,
                "live_canonical_frac": live / (kms * 1e-3) / 1e12 / peak,
                "traffic": prof,
                "peak_source": "measured DFMA probe (mf_fp64_probe) "
                               "in this run",
                "kernel_ms": kms,
                "algorithmic_flops": canonical,
                "executed_flops": executed,
                "executed_tflops": achieved,
                "executed_frac": achieved / peak}
        cfgk = CONFIGS[name]
        if cfgk[0] == 3 and cfgk[6] == "hex" and cfgk[7] == 2:
            # k_hex2 issues 3 NO + 9 NO + 5 NO^2 + 12 NO^3 FP64 warp
            # instructions per full event (mf_hex2.cu event_full2: 405 for
            # NO = 3); the DFMA probe's peak is 64 flops per warp
            # instruction.  This is the share of the FP64 pipe's issue
            # slots the full events alone fill (ncu's FP64 pipe % of the
            # same launch is a few points higher: classification, axes).
            no = 2 if cfgk[8] == "gauss2" else 3
            per_ev = 12 * no + 5 * no * no + 12 * no ** 3
            rate = int(cnt[N.CNT_EV_FULL]) * per_ev / (kms * 1e-3)
            roof["fp64_issue_frac_full_events"] = rate / (peak * 1e12 / 64)
            roof["fp64_warp_instr_per_full_event"] = per_ev
    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_all, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic (seeded jittered-lattice Delaunay mesh)"
                 if CONFIGS[name][6] == "delaunay" else
                 "synthetic (structured mesh, reference-realisable "
                 "stand-in)"),
        "kernel_ms_per_step": statistics.mean(kern_ms),
        "config": config_json(name, mesh, space, world, slab,
                              args.strategy),
        "events": int(cnt[N.CNT_EVENTS]), "pairs": pairs_all,
        "event_classes": {"upper_plateau": int(cnt[N.CNT_EV_UPPER]),
                          "lmax_plateau": int(cnt[N.CNT_EV_PLATEAU]),
                          "lmax_dead": int(cnt[N.CNT_EV_DEAD]),
                          "lmax_full": int(cnt[N.CNT_EV_FULL])},
        "counters": [int(c) for c in cnt],
        "roofline": roof,
        "gpu_launches": int(args.steps * n_launch),
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if (world == 1 and not args.no_e2e and args.strategy == "general"
            and mesh.kind in ("tri", "quad", "hex")
            and not getattr(mesh, "unstructured", False)):
        # the reference's DEFAULT path on structured meshes is the
        # offset-blocked strategy (assemble(strategy="auto"),
        # assembly.py:448-473): the like-for-like end-to-end comparison
        # with the reference arm's cpu_baseline.default_path
        from paper_2101_08825_b200 import AssemblyConfig
        auto = AssemblyConfig(L_max=cfg.L_max, outer_rule=cfg.outer_rule,
                              inner_rule=cfg.inner_rule, strategy="auto")
        B = assemble(mesh, space, kp, auto, device=dev)
        del B
        torch.cuda.synchronize()
        ts = []
        for _ in range(2):
            t = time.perf_counter()
            B = assemble(mesh, space, kp, auto, device=dev)
            _ = B.vals[-1]
            ts.append(time.perf_counter() - t)
            del B
        line["e2e_default_path"] = {
            "value": pairs_all / min(ts), "unit": "pairs/s",
            "seconds_per_assembly": min(ts),
            "path": "assemble(strategy='auto') -> GPU offset-blocked "
                    "(mf_offset_blocks + gather), host in, host out"}
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_sample(name, mesh, space, kp, cfg,
                                          budget_s=args.cpu_budget)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def launches_per_group(mesh):
    """Kernel launches per non-empty colour group of mf_general_core:
    tets run two parity launches + the A22 fold (mf_tet.cu), Delaunay
    triangles row_period row-class launches + the fold (k_tri_u), the
    other kernels one launch."""
    if mesh.kind == "tet":
        return 3
    if getattr(mesh, "unstructured", False):
        return int(mesh.row_period) + 1
    return 1


def ctx_nnz(mesh, space, kp, cfg):
    from paper_2101_08825_b200.assembly import HostPattern, pattern_halfwidth
    K, _ = pattern_halfwidth(mesh, kp, cfg, space.degree)
    return int(HostPattern(space, K, allocate=False).rowptr[-1])


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def load_traffic(name):
    """dram bytes per launch of the dominant kernel from profiles/."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(name)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="R4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--strategy", default="general",
                    choices=["general", "blocked"],
                    help="general = per-pair Algorithm 1 (headline); "
                         "blocked = the reference's offset-blocked default")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-step-budget", type=float, default=6.0,
                    help="--impl reference: seconds of CPU work per timed "
                         "step (warm-up steps use 1 s)")
    ap.add_argument("--no-default-path", action="store_true",
                    help="--impl reference: skip timing the reference "
                         "default (blocked) assemble()")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
