"""The C-ABI library loads and exports every symbol the header declares."""

import os
import re

from conftest import ROOT


def _header_functions():
    src = open(os.path.join(ROOT, "include", "mollifem_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_2101_08825_b200 import _native as N
    L = N.load_library()
    names = _header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(N.EXPORTED)
    assert L.mf_abi_version() == N.ABI_VERSION == 3


def test_library_is_sm100a_only():
    import subprocess
    from paper_2101_08825_b200 import _native as N
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out


def test_compute_calls_fail_loudly_without_gpu():
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2101_08825_b200 import _native as N
    with pytest.raises(RuntimeError, match="CUDA device"):
        N.lib()


def test_overflow_counter_raises():
    """A kernel that reports dropped work (MF_CNT_OVERFLOW) makes finish()
    raise instead of returning an incomplete matrix."""
    import numpy as np
    import pytest
    from paper_2101_08825_b200 import _native as N
    from paper_2101_08825_b200.assembly import check_counters
    c = np.zeros(N.MF_NCOUNTERS, np.int64)
    check_counters(c)
    c[N.CNT_OVERFLOW] = 1
    with pytest.raises(RuntimeError, match="overflow"):
        check_counters(c)
