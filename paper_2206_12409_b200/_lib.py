"""ctypes declarations of include/vsie_coupling.h (argument marshalling only).

The shared library is built in-tree by ``paper_2206_12409_b200._build``.  If
it is missing the import fails loudly: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libvsie_coupling.so")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
HEADER = os.path.join(INCLUDE, "vsie_coupling.h")

VSIE_OK = 0
VSIE_WARN_NOT_CONVERGED = 1
OPS = {"N": 0, "T": 1, "C": 2}


class vsie_grid(C.Structure):
    _fields_ = [("n", C.c_int32 * 3), ("h", C.c_double * 3), ("origin", C.c_double * 3)]


class vsie_mesh(C.Structure):
    _fields_ = [("n_vertices", C.c_int64), ("xyz", C.c_void_p), ("n_triangles", C.c_int64), ("tri", C.c_void_p)]


class vsie_build_opts(C.Structure):
    _fields_ = [("max_rank", C.c_int32), ("max_sweeps", C.c_int32), ("oversample", C.c_int32),
                ("direct_svd_max", C.c_int32), ("heldout", C.c_int32), ("nrhs_max", C.c_int32),
                ("seed", C.c_uint64), ("scale_re", C.c_double), ("scale_im", C.c_double),
                ("rank", C.c_int32), ("world", C.c_int32), ("loopback", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("device", C.c_int32), ("verbose", C.c_int32),
                ("test_moment", C.c_int32), ("ipc_name", C.c_char_p), ("quad_rule", C.c_int32)]


class vsie_info(C.Structure):
    _fields_ = [("n", C.c_int32 * 3), ("m", C.c_int64), ("ranks", (C.c_int32 * 3) * 3),
                ("core_bytes", C.c_int64), ("compression_num", C.c_int64), ("compression_den", C.c_int64),
                ("entries_evaluated", C.c_int64), ("sweeps", C.c_int32 * 3), ("heldout_err", C.c_double * 3),
                ("build_s", C.c_double), ("build_entry_s", C.c_double), ("build_factor_s", C.c_double),
                ("build_maxvol_s", C.c_double), ("slab", C.c_int32 * 2), ("cols", C.c_int64 * 2),
                ("world", C.c_int32), ("rank", C.c_int32), ("loopback", C.c_int32), ("k0", C.c_double),
                ("apply_launches", C.c_int64), ("apply_calls", C.c_int64), ("test_moment", C.c_int32),
                ("pair_schedule", C.c_int32), ("quad_rule", C.c_int32)]


class vsie_timer(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("total_ms", C.c_double),
                ("bytes_per_launch", C.c_int64), ("flops_per_launch", C.c_int64)]


class vsie_trace(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("chi", C.c_int32), ("call", C.c_int32), ("t0_ms", C.c_double),
                ("t1_ms", C.c_double)]


class vsie_farnear_opts(C.Structure):
    _fields_ = [("max_rank", C.c_int32), ("scale_re", C.c_double), ("scale_im", C.c_double), ("device", C.c_int32),
                ("verbose", C.c_int32)]


class vsie_farnear_info(C.Structure):
    _fields_ = [("m_near", C.c_int64), ("m_far", C.c_int64), ("rank", C.c_int32), ("stop", C.c_int32),
                ("est_err", C.c_double), ("frob", C.c_double), ("min_distance", C.c_double),
                ("max_edge", C.c_double), ("k0", C.c_double), ("build_s", C.c_double),
                ("entries_evaluated", C.c_int64), ("factor_bytes", C.c_int64), ("apply_calls", C.c_int64)]


class vsie_hybrid_info(C.Structure):
    _fields_ = [("m_far", C.c_int64), ("m_near", C.c_int64), ("n_body", C.c_int64), ("n", C.c_int64),
                ("matvecs", C.c_int64)]


class vsie_gmres_info(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("restarts", C.c_int32), ("converged", C.c_int32),
                ("rel_residual", C.c_double), ("seconds", C.c_double), ("matvec_seconds", C.c_double)]


class vsie_farfar_info(C.Structure):
    _fields_ = [("m", C.c_int64), ("tile", C.c_int32), ("tiles", C.c_int64), ("matrix_bytes", C.c_int64),
                ("near_pairs", C.c_int64), ("build_s", C.c_double), ("k0", C.c_double), ("apply_calls", C.c_int64)]


HANDLE = C.c_void_p
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)

_SIGS = {
    "vsie_abi_version": (C.c_int32, []),
    "vsie_set_allocator": (C.c_int32, [ALLOC_FN, FREE_FN, C.c_void_p]),
    "vsie_build_opts_default": (None, [C.POINTER(vsie_build_opts)]),
    "vsie_status_string": (C.c_char_p, [C.c_int32]),
    "vsie_last_error_message": (C.c_char_p, []),
    "vsie_nccl_unique_id": (C.c_int32, [C.c_void_p]),
    "vsie_slab_partition": (C.c_int32, [C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int64)]),
    "vsie_coupling_build": (C.c_int32, [C.POINTER(vsie_grid), C.POINTER(vsie_mesh), C.c_int32, C.c_double,
                                        C.c_double, C.POINTER(vsie_build_opts), C.POINTER(HANDLE)]),
    "vsie_coupling_import_cores": (C.c_int32, [C.POINTER(vsie_grid), C.POINTER(vsie_mesh), C.c_int32, C.c_double,
                                               C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                                               C.POINTER(vsie_build_opts), C.POINTER(HANDLE)]),
    "vsie_coupling_export_cores": (C.c_int32, [HANDLE, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_int64)]),
    "vsie_coupling_round": (C.c_int32, [HANDLE, C.c_double]),
    "vsie_coupling_apply": (C.c_int32, [HANDLE, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "vsie_coupling_apply_host": (C.c_int32, [HANDLE, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]),
    "vsie_coupling_entries": (C.c_int32, [HANDLE, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "vsie_coupling_tt_eval": (C.c_int32, [HANDLE, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "vsie_coupling_supercore": (C.c_int32, [HANDLE, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                            C.c_int32, C.c_void_p, C.c_void_p]),
    "vsie_coupling_info": (C.c_int32, [HANDLE, C.POINTER(vsie_info)]),
    "vsie_coupling_set_timing": (C.c_int32, [HANDLE, C.c_int32]),
    "vsie_coupling_timers": (C.c_int32, [HANDLE, C.POINTER(vsie_timer), C.c_int32, C.POINTER(C.c_int32)]),
    "vsie_coupling_apply_pair": (C.c_int32, [HANDLE, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                             C.c_void_p]),
    "vsie_coupling_apply_pair_host": (C.c_int32, [HANDLE, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]),
    "vsie_coupling_apply_pwl": (C.c_int32, [C.POINTER(HANDLE), C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                            C.c_void_p]),
    "vsie_coupling_apply_pair_pwl": (C.c_int32, [C.POINTER(HANDLE), C.c_void_p, C.c_void_p, C.c_void_p,
                                                 C.c_void_p, C.c_int32, C.c_void_p]),
    "vsie_coupling_configure": (C.c_int32, [HANDLE, C.c_int32, C.c_int32]),
    "vsie_coupling_trace": (C.c_int32, [HANDLE, C.POINTER(vsie_trace), C.c_int32, C.POINTER(C.c_int32)]),
    "vsie_coupling_destroy": (None, [HANDLE]),
    # include/vsie_farnear.h
    "vsie_farnear_opts_default": (None, [C.POINTER(vsie_farnear_opts)]),
    "vsie_farnear_build": (C.c_int32, [C.POINTER(vsie_mesh), C.c_int32, C.POINTER(vsie_mesh), C.c_int32, C.c_double,
                                       C.c_double, C.POINTER(vsie_farnear_opts), C.POINTER(HANDLE)]),
    "vsie_farnear_entries": (C.c_int32, [HANDLE, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "vsie_farnear_apply": (C.c_int32, [HANDLE, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "vsie_farnear_apply_pair": (C.c_int32, [HANDLE, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vsie_farnear_export": (C.c_int32, [HANDLE, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vsie_farnear_get_info": (C.c_int32, [HANDLE, C.POINTER(vsie_farnear_info)]),
    "vsie_farnear_destroy": (None, [HANDLE]),
    # include/vsie_farfar.h
    "vsie_farfar_build": (C.c_int32, [C.POINTER(vsie_mesh), C.c_int32, C.c_double, C.c_double, C.c_double, C.c_int32,
                                      C.POINTER(HANDLE)]),
    "vsie_farfar_entries": (C.c_int32, [HANDLE, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "vsie_farfar_apply": (C.c_int32, [HANDLE, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    "vsie_farfar_export": (C.c_int32, [HANDLE, C.c_void_p]),
    "vsie_farfar_get_info": (C.c_int32, [HANDLE, C.POINTER(vsie_farfar_info)]),
    "vsie_hybrid_create": (C.c_int32, [HANDLE, HANDLE, HANDLE, HANDLE, HANDLE, C.c_void_p, C.POINTER(HANDLE)]),
    "vsie_hybrid_matvec": (C.c_int32, [HANDLE, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vsie_hybrid_gmres": (C.c_int32, [HANDLE, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_double,
                                      C.c_void_p, C.POINTER(vsie_gmres_info), C.c_void_p]),
    "vsie_hybrid_get_info": (C.c_int32, [HANDLE, C.POINTER(vsie_hybrid_info)]),
    "vsie_hybrid_destroy": (None, [HANDLE]),
    "vsie_farfar_destroy": (None, [HANDLE]),
}


def header_symbols(paths=None):
    """Function names declared in include/*.h."""
    if paths is None:
        paths = sorted(os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE) if f.endswith(".h"))
    txt = "".join(open(p).read() for p in paths)
    return sorted(set(re.findall(r"\b(vsie_[a-z_]+)\s*\(", txt))
                  - {"vsie_coupling_t", "vsie_farnear_t", "vsie_farfar_t", "vsie_hybrid_t"})


class VsieError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{status}: {msg}")
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2206_12409_b200._build` "
                "(there is no CPU fallback)")
        # RTLD_NOW: an unresolved symbol fails the load here, not at first call
        L = C.CDLL(LIB_PATH, mode=os.RTLD_NOW | os.RTLD_LOCAL)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int, allow_warn: bool = False) -> int:
    if status == VSIE_OK or (allow_warn and status > 0):
        return status
    L = lib()
    raise VsieError(L.vsie_status_string(status).decode(), L.vsie_last_error_message().decode())
