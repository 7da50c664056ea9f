"""The reference-side binding has the reference hooks' exact signatures
(no GPU needed: signatures only)."""

import inspect

import pytest


def _reference():
    import bench
    mf = bench.ref_import()
    if mf is None:
        pytest.skip("reference not installed under baseline/_ref")
    return mf


def _names(f):
    return [p for p in inspect.signature(f).parameters if p != "device"]


def test_general_core_signature():
    _reference()
    from mollifem import _kernels as K
    from paper_2101_08825_b200 import refbind
    ref = getattr(K._general_core, "py_func", K._general_core)
    assert _names(refbind.general_core) == _names(ref)


def test_run_general_signature():
    _reference()
    from mollifem import assembly as RA
    from paper_2101_08825_b200 import refbind
    assert _names(refbind.run_general) == _names(RA._run_general)
