"""SparseMatrix / host-transfer contract details."""

import threading

import numpy as np
import pytest

from conftest import Golden

pytestmark = pytest.mark.gpu


def test_mirrored_host_values_are_read_only():
    """While a device copy exists the host vals cannot be edited in place
    (a stale device copy would silently feed matvec/diag/solve); assigning
    a new array drops the device copy and the next device method uses it."""
    from paper_2101_08825_b200 import assemble
    g = Golden("quad_q1_lmax3")
    mesh, space, kp, cfg = g.build()
    A = assemble(mesh, space, kp, cfg)
    with pytest.raises(ValueError):
        A.vals[0] = 1.0
    d0 = A.diag()
    v = A.vals.copy()
    v[:] = 0.0
    A.vals = v
    assert np.all(A.diag() == 0.0)
    A.vals = 2.0 * g["vals"]
    assert np.allclose(A.diag(), 2.0 * d0, rtol=1e-12, atol=0.0)
    B = A.copy_pattern()            # host-only: writable, as the reference
    B.vals[:] = 1.0


def test_concurrent_host_copies_do_not_interleave():
    """Two threads copying large device arrays to the host at once share
    the per-device staging ring; the lock keeps each result intact."""
    import torch
    from paper_2101_08825_b200.assembly import _STREAM_MIN_BYTES, _d2h
    n = _STREAM_MIN_BYTES // 8 + 12345
    a = torch.arange(n, dtype=torch.float64, device="cuda")
    b = -torch.arange(n, dtype=torch.float64, device="cuda")
    out = {}

    def run(key, t):
        out[key] = _d2h(t)

    th = [threading.Thread(target=run, args=("a", a)),
          threading.Thread(target=run, args=("b", b))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    ref = np.arange(n, dtype=np.float64)
    assert np.array_equal(out["a"], ref)
    assert np.array_equal(out["b"], -ref)
