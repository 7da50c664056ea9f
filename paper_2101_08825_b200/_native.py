"""ctypes binding of libmollifem_b200.so (include/mollifem_b200.h).

PyTorch provides device memory and streams only; every tensor crosses the
boundary as a raw pointer.  There is no fallback: if the library or a CUDA
device is missing, `lib()` raises.
"""

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MF_LIB_PATH") or os.path.join(
    _HERE, "_lib", "libmollifem_b200.so")

MF_NCOUNTERS = 10
CNT_EVENTS, CNT_PAIRS, CNT_EV_UPPER, CNT_EV_PLATEAU, CNT_EV_DEAD, \
    CNT_EV_FULL, CNT_OVERFLOW = range(7)
ABI_VERSION = 3
FLAG_FORCE_GENERIC = 1
FLAG_NO_SHORTCUTS = 2
FLAG_ELEMENT_THREADS = 4
FLAG_HEX_LEVELS = 8


class MfMesh(C.Structure):
    _fields_ = [("dim", C.c_int32), ("degree", C.c_int32),
                ("n_elem", C.c_int64), ("nv_max", C.c_int32),
                ("nloc_max", C.c_int32), ("elem_kind", C.c_void_p),
                ("elem_coords", C.c_void_p), ("elem_lo", C.c_void_p),
                ("elem_hi", C.c_void_p), ("elem_dofs", C.c_void_p),
                ("elem_cell", C.c_void_p), ("cell_ptr", C.c_void_p),
                ("ncx", C.c_int32), ("ncy", C.c_int32), ("ncz", C.c_int32),
                ("kinds_present", C.c_int32), ("layout", C.c_int32),
                ("row_period", C.c_int32)]


class MfRules(C.Structure):
    _fields_ = [("nq_box_out", C.c_int32), ("nq_box_in", C.c_int32),
                ("nq_tri_out", C.c_int32), ("nq_tri_in", C.c_int32)] + [
        (n, C.c_void_p) for n in (
            "box_out_pts", "box_out_w", "box_in_pts", "box_in_w",
            "tri_out_pts", "tri_out_w", "tri_in_pts", "tri_in_w",
            "phi_box_in", "phi_tri_in")] + [
        ("n1d_box_out", C.c_int32), ("n1d_box_in", C.c_int32)] + [
        (n, C.c_void_p) for n in ("box_out_x1d", "box_out_w1d",
                                  "box_in_x1d", "box_in_w1d")]


class MfKernel(C.Structure):
    _fields_ = [("delta", C.c_double), ("eps", C.c_double),
                ("cde", C.c_double), ("L_min", C.c_int32),
                ("L_max", C.c_int32)]


class MfPattern(C.Structure):
    _fields_ = [("NX", C.c_int32), ("NY", C.c_int32), ("NZ", C.c_int32),
                ("K", C.c_int32), ("n", C.c_int64), ("rowptr", C.c_void_p)]


# name -> (restype, argtypes)
_P = C.c_void_p
_SIGS = {
    "mf_count_candidates": (C.c_int, [C.POINTER(MfMesh), _P, C.c_int64, _P,
                                      C.c_int32, C.c_double, _P, _P]),
    "mf_fill_candidates": (C.c_int, [C.POINTER(MfMesh), _P, C.c_int64, _P,
                                     C.c_int32, C.c_double, _P, _P, _P]),
    "mf_scan_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "mf_exclusive_scan": (C.c_int, [_P, C.c_int64, _P, _P, C.c_size_t, _P]),
    "mf_general_workspace_bytes": (C.c_size_t, [C.POINTER(MfMesh),
                                                C.POINTER(MfRules),
                                                C.c_int64]),
    "mf_general_core": (C.c_int, [C.POINTER(MfMesh), C.POINTER(MfRules),
                                  C.POINTER(MfKernel), C.POINTER(MfPattern),
                                  _P, _P, _P, C.c_int32, C.c_int32,
                                  C.c_double, _P, _P, C.c_int32, _P,
                                  C.c_size_t, _P]),
    "mf_general_core_lists": (C.c_int, [C.POINTER(MfMesh),
                                        C.POINTER(MfRules),
                                        C.POINTER(MfKernel),
                                        C.POINTER(MfPattern), _P, C.c_int64,
                                        _P, _P, C.c_double, _P, _P,
                                        C.c_int32, _P]),
    "mf_offset_block_count": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "mf_offset_blocks_workspace_bytes": (C.c_size_t, [C.POINTER(MfRules),
                                                      C.c_int64]),
    "mf_offset_blocks": (C.c_int, [C.POINTER(MfMesh), C.POINTER(MfRules),
                                   C.POINTER(MfKernel), C.c_int32, C.c_int32,
                                   _P, C.c_int32, C.c_double, _P, _P, _P,
                                   C.c_int32, _P, C.c_size_t, _P]),
    "mf_scatter_offset_blocks": (C.c_int, [C.POINTER(MfMesh),
                                           C.POINTER(MfPattern), C.c_int32,
                                           C.c_int32, _P, _P, _P, _P, _P, _P,
                                           _P, _P, C.c_int32, C.c_double, _P,
                                           _P, _P]),
    "mf_gather_table_doubles": (C.c_int64, [C.c_int32, C.c_int32,
                                            C.c_int32]),
    "mf_offset_block_a22": (C.c_int, [C.POINTER(MfMesh), C.c_int32,
                                      C.c_int32, C.c_int32, _P, _P, _P, _P,
                                      _P, _P, _P]),
    "mf_gather_offset_blocks": (C.c_int, [C.POINTER(MfMesh),
                                          C.POINTER(MfPattern), C.c_int32,
                                          C.c_int32, C.c_int32, _P, _P,
                                          C.c_int64, C.c_int64, C.c_double,
                                          _P, _P]),
    "mf_scale": (C.c_int, [_P, C.c_int64, C.c_double, _P]),
    "mf_asymmetry_inf": (C.c_int, [C.POINTER(MfPattern), _P, _P, _P]),
    "mf_asymmetry_inf_rows": (C.c_int, [C.POINTER(MfPattern), _P, C.c_int64,
                                        C.c_int64, _P, _P]),
    "mf_norm_inf": (C.c_int, [C.POINTER(MfPattern), _P, _P, _P]),
    "mf_matvec": (C.c_int, [C.POINTER(MfPattern), _P, _P, _P, _P]),
    "mf_diag": (C.c_int, [C.POINTER(MfPattern), _P, _P, _P]),
    "mf_symmetrize": (C.c_int, [C.POINTER(MfPattern), _P, _P]),
    "mf_fill_cols": (C.c_int, [C.POINTER(MfPattern), _P, _P]),
    "mf_load_scatter": (C.c_int, [C.POINTER(MfMesh), _P, _P, C.c_int32, _P,
                                  _P, _P, C.c_int32, C.c_int32, _P, _P]),
    "mf_vec_workspace_bytes": (C.c_size_t, []),
    "mf_cg_matvec_dot": (C.c_int, [C.POINTER(MfPattern), _P, _P, _P, _P, _P,
                                   _P, _P]),
    "mf_cg_update": (C.c_int, [C.c_int64, C.c_double, _P, _P, _P, _P, _P, _P,
                               _P, _P, _P]),
    "mf_cg_direction": (C.c_int, [C.c_int64, C.c_double, _P, _P, _P]),
    "mf_jacobi_inverse": (C.c_int, [C.c_int64, _P, _P, _P, _P, _P, _P]),
    "mf_gather_diff": (C.c_int, [C.c_int64, _P, _P, _P, _P, _P]),
    "mf_scatter_values": (C.c_int, [C.c_int64, _P, _P, _P, _P]),
    "mf_sum_ordered": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p),
                                 C.c_int64, C.c_double, _P, _P]),
    "mf_row_touched": (C.c_int, [C.POINTER(MfPattern), _P, _P, _P]),
    "mf_axpby": (C.c_int, [C.c_int64, C.c_double, _P, C.c_double, _P, _P,
                           _P]),
    "mf_matvec_rows": (C.c_int, [C.POINTER(MfPattern), _P, _P, C.c_int64,
                                 C.c_int64, _P, _P]),
    "mf_fp64_probe": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, _P]),
    "mf_fp64_probe_flops": (C.c_double, [C.c_int64, C.c_int32, C.c_int32]),
    "mf_last_error": (C.c_char_p, []),
    "mf_abi_version": (C.c_int, []),
}

EXPORTED = tuple(_SIGS)
_lib = None


def load_library():
    """dlopen the library and bind every symbol (no CUDA device needed)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA library {LIB_PATH} is missing; run "
                "__graft_entry__.build() (make -C paper_2101_08825_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def lib():
    """Library handle for compute calls; requires a CUDA device."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2101_08825_b200 needs a CUDA device "
                           "(B200, sm_100a); there is no CPU fallback")
    return load_library()


def check(rc, what):
    if rc != 0:
        msg = load_library().mf_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed (code {rc}): {msg}")


def ptr(t):
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_ptr(stream=None, device=None):
    """cudaStream_t of `stream`, else of the current stream of `device`
    (default: the current device)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return C.c_void_p(s.cuda_stream)
