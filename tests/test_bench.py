"""bench.py bookkeeping that does not need a GPU."""

import numpy as np
import pytest


@pytest.mark.parametrize("name", ["R1", "R4-small"])
def test_pair_table_matches_oracle(name, oracle_lib):
    import bench
    mesh, space, kp, cfg = bench.build_problem(name)
    n = mesh.n_elements
    ptr, _ = oracle_lib.candidates(mesh, kp.delta + kp.eps, np.arange(n),
                                   np.ones(n, np.uint8))
    assert int(ptr[-1]) == bench.PAIRS[name]


def test_flop_model_canonical_matches_survey():
    """R1 total 4.77e9, R4 2.36e14 canonical flops."""
    import bench
    from paper_2101_08825_b200 import _native as N
    c = np.zeros(8, np.int64)
    c[N.CNT_EVENTS], c[N.CNT_PAIRS] = 5800432, 462400
    _, canon = bench.flop_model("R1", c)
    assert abs(canon / 4.77e9 - 1) < 0.01
    c[N.CNT_EVENTS], c[N.CNT_PAIRS] = 9994768232, 1382469544
    _, canon = bench.flop_model("R4", c)
    assert abs(canon / 2.36e14 - 1) < 0.01


def test_reference_arm_runs_the_reference():
    """--impl reference times the unmodified reference (numba, baseline/_ref)
    and the reference default (blocked) path, on the host cores."""
    import json
    import os
    import subprocess
    import sys
    import bench
    if bench.ref_import() is None:
        pytest.skip("reference not installed under baseline/_ref")
    r = subprocess.run(
        [sys.executable, os.path.join(bench.ROOT, "bench.py"), "--impl",
         "reference", "--config", "R1", "--steps", "1", "--warmup", "1",
         "--ref-step-budget", "0.5"], capture_output=True, text=True,
        timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1
    assert cb["value"] == line["value"] > 0
    d = cb["default_path"]
    assert d["workload"] == "R1" and d["pairs"] == bench.PAIRS["R1"]
    assert d["events"] > 0 and d["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
