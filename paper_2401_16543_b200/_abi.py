"""ctypes view of the C-ABI in include/kfvm_b200.h (plumbing only).

The product path is libkfvm_b200.so, built in-tree by `make` (see
__graft_entry__.build()).  Loading fails loudly when the library is missing:
there is no Python or CPU fallback for the stage update.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KFVM_LIB") or os.path.join(_HERE, "libkfvm_b200.so")

KFVM_OK, KFVM_ERR_CONFIG, KFVM_ERR_RUNTIME, KFVM_ERR_DEVICE = 0, 1, 2, 3
BC_PERIODIC, BC_OUTFLOW, BC_REFLECTING, BC_DIRICHLET, BC_SLIT = 0, 1, 2, 3, 4
RIEMANN_HLLC, RIEMANN_HLL = 0, 1
IC_FOURIER, IC_VORONOI, IC_FOURIER_SPHERE, IC_UNIFORM, IC_VORTEX, IC_DENSITY_WAVE = range(6)


class KfvmTable(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("radius", C.c_int), ("n_stencils", C.c_int),
        ("n_points", C.c_int), ("n_alpha", C.c_int), ("n_full", C.c_int),
        ("total_cells", C.c_int),
        ("size", C.c_int * 8), ("degree", C.c_int * 8), ("cell_offset", C.c_int * 8),
        ("offsets", C.POINTER(C.c_int)), ("gather", C.POINTER(C.c_int)),
        ("alpha", C.POINTER(C.c_int)),
        ("face", C.POINTER(C.c_double)), ("deriv", C.POINTER(C.c_double)),
        ("gamma_lin", C.POINTER(C.c_double)), ("face_weights", C.POINTER(C.c_double)),
        ("points", C.POINTER(C.c_double)), ("gl_nodes", C.POINTER(C.c_double)),
        ("gl_weights", C.POINTER(C.c_double)),
        ("ell_over_delta", C.c_double), ("hash", C.c_uint64),
    ]


class KfvmConfig(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("radius", C.c_int), ("nx", C.c_int), ("ny", C.c_int),
        ("nz", C.c_int), ("bc", C.c_int), ("riemann", C.c_int),
        ("dx", C.c_double), ("gamma", C.c_double), ("cfl", C.c_double),
        ("eps", C.c_double), ("kappa", C.c_double), ("flattener_kf", C.c_double),
        ("kxrcf", C.c_int), ("kxrcf_m", C.c_double),
        ("integrator", C.c_int), ("atol", C.c_double), ("rtol", C.c_double),
        ("safety", C.c_double), ("dt_min", C.c_double), ("dt_max", C.c_double),
        ("viscous", C.c_int), ("reynolds", C.c_double), ("prandtl", C.c_double),
        ("mach", C.c_double), ("inv_froude2", C.c_double),
        ("bc_per_side", C.c_int), ("bc_side", C.c_int * 6),
        ("bc_state", (C.c_double * 5) * 6), ("slit_center", (C.c_double * 2) * 6),
        ("slit_radius", C.c_double * 6),
    ]


class KfvmIcParams(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("n_modes", C.c_int), ("n_regions", C.c_int),
        ("seed", C.c_uint64), ("origin", C.c_double * 3), ("value", C.c_double * 5),
    ]


class KfvmDist(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("device", C.c_int),
                ("nccl_id", C.c_ubyte * 128)]


EXPORTS = [
    # (name, restype, argtypes)
    ("kfvm_table_build", C.c_int, [C.c_int, C.c_int, C.c_double, C.POINTER(C.POINTER(KfvmTable))]),
    ("kfvm_table_free", None, [C.POINTER(KfvmTable)]),
    ("kfvm_config_defaults", None, [C.POINTER(KfvmConfig), C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int]),
    ("kfvm_ic_generate", C.c_int, [C.POINTER(KfvmConfig), C.POINTER(KfvmIcParams), C.c_int,
                                   C.c_int, C.c_int, C.c_void_p]),
    ("kfvm_nccl_unique_id", C.c_int, [C.c_void_p]),
    ("kfvm_loopback_id", C.c_int, [C.c_void_p]),
    ("kfvm_slab_range", None, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("kfvm_gpu_create", C.c_int, [C.POINTER(KfvmConfig), C.POINTER(KfvmTable), C.POINTER(KfvmDist),
                                  C.POINTER(C.c_void_p)]),
    ("kfvm_gpu_destroy", None, [C.c_void_p]),
    ("kfvm_gpu_set_state", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kfvm_gpu_get_state", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kfvm_gpu_set_state_async", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kfvm_gpu_get_state_async", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kfvm_gpu_set_state_device", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kfvm_gpu_get_state_device", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kfvm_gpu_rhs", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kfvm_gpu_states", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kfvm_gpu_select_dt", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("kfvm_gpu_kxrcf_flags", C.c_int, [C.c_void_p, C.c_void_p]),
    ("kfvm_gpu_step_stats", C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("kfvm_gpu_stage", C.c_int, [C.c_void_p, C.c_int, C.c_double]),
    ("kfvm_gpu_step", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("kfvm_gpu_run", C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    ("kfvm_gpu_run_async", C.c_int, [C.c_void_p, C.c_int]),
    ("kfvm_gpu_sync", C.c_int, [C.c_void_p]),
    ("kfvm_gpu_dt_sequence", C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    ("kfvm_gpu_stream", C.c_void_p, [C.c_void_p]),
    ("kfvm_gpu_launch_count", C.c_longlong, [C.c_void_p]),
    ("kfvm_gpu_set_option", C.c_int, [C.c_void_p, C.c_char_p, C.c_longlong]),
    ("kfvm_gpu_kernel_times", C.c_int, [C.c_void_p] + [C.POINTER(C.c_double)] * 4),
    ("kfvm_gpu_last_error", C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    ("kfvm_gpu_ic_generate", C.c_int, [C.c_void_p, C.POINTER(KfvmIcParams)]),
    ("kfvm_fp64_peak", C.c_int, [C.POINTER(C.c_double)] * 3),
    ("kfvm_phase_cycles", C.c_int, [C.POINTER(C.c_ulonglong), C.c_int]),
    ("kfvm_gpu_advance_to", C.c_int, [C.c_void_p, C.c_double, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_double)]),
]

_lib = None


def lib() -> C.CDLL:
    """Load libkfvm_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                "there is no fallback path")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, res, args in EXPORTS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
