"""Shared fixtures: golden cases, host-layer builders, oracle access."""

import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers",
                            "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden_names():
    """Structured-mesh fixtures of make_golden.py (the Delaunay fixtures of
    make_golden_delaunay.py have their own tests, test_delaunay.py)."""
    return sorted(os.path.basename(p)[:-4]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if not os.path.basename(p).startswith("delaunay_"))


class Golden:
    """One golden case: reference outputs + our host-layer inputs."""

    def __init__(self, name):
        self.name = name
        self.z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
        self.meta = json.loads(str(self.z["meta"]))

    def __getitem__(self, k):
        return self.z[k]

    def __contains__(self, k):
        return k in self.z.files

    def build(self):
        from paper_2101_08825_b200 import (AssemblyConfig, FESpace,
                                           KernelParams, build_mesh)
        m = self.meta
        kp = KernelParams(m["dim"], m["delta"], m["eps"], m["kappa"])
        mesh = build_mesh(m["dim"], m["omega"], m["h"],
                          m["delta"] + m["eps"], m["kind"])
        space = FESpace(mesh, m["degree"])
        cfg = AssemblyConfig(L_min=m["L_min"], L_max=m["L_max"],
                             outer_rule=m["outer_rule"],
                             inner_rule=m["inner_rule"], strategy="general")
        return mesh, space, kp, cfg


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


def rel_frob(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
