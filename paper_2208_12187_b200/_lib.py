"""ctypes binding of libjfb200.so (include/jf.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels.  There is no
CPU fallback — if the library cannot be loaded, every call raises."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libjfb200.so")

JF_MAX_N = 16
JF_COMM_HANDLE_BYTES = 256
JF_TRACE_FIELDS = 12

# jf_model
LINEAR, EXP_DECAY, GAUSS1D, GAUSS2D_ROT, GAUSS2D_ROT_X2 = range(5)
MODEL_IDS = {"linear": LINEAR, "exp_decay": EXP_DECAY, "gauss1d": GAUSS1D,
             "gauss2d_rot": GAUSS2D_ROT, "gauss2d_rot_x2": GAUSS2D_ROT_X2}
# jf_xscale / jf_solver / jf_policy
XSCALE_JAC, XSCALE_ONES, XSCALE_ARRAY = range(3)
SOLVE_AUTO, SOLVE_GRAM, SOLVE_TSQR = range(3)
POLICY_SPECULATIVE, POLICY_CONSERVATIVE = range(2)
# errors
EINVAL, EINFEASIBLE, ENONFINITE, ECUDA, ECOMM, ENOMEM = -1, -2, -3, -4, -5, -6


class jf_opts(C.Structure):
    _fields_ = [
        ("ftol", C.c_double), ("xtol", C.c_double), ("gtol", C.c_double),
        ("max_nfev", C.c_int32), ("x_scale_mode", C.c_int32),
        ("x_scale", C.POINTER(C.c_double)),
        ("solver", C.c_int32), ("policy", C.c_int32),
        ("grid_w", C.c_int64), ("grid_h", C.c_int64), ("grid_row0", C.c_int64),
        ("t0", C.c_double), ("dt", C.c_double), ("index0", C.c_int64),
        ("sigma", C.c_void_p),
        ("device", C.c_int32), ("inputs_on_device", C.c_int32),
        ("stream", C.c_void_p), ("comm", C.c_void_p),
        ("use_graph", C.c_int32), ("trace_cap", C.c_int32),
        ("trace", C.POINTER(C.c_double)),
        ("m_global", C.c_int64),
        ("capacity", C.c_int64), ("flags", C.c_int32), ("pad_opts_", C.c_int32),
        ("x_host", C.POINTER(C.c_double)),
    ]


FLAG_ALT_COORDS = 1
FLAG_BATCH_SHARED_Y = 2


class jf_batch_result(C.Structure):
    _fields_ = [("x", C.c_double * JF_MAX_N), ("cost", C.c_double), ("optimality", C.c_double),
                ("status", C.c_int32), ("nfev", C.c_int32), ("njev", C.c_int32), ("nit", C.c_int32)]


class jf_result(C.Structure):
    _fields_ = [
        ("x", C.c_double * JF_MAX_N), ("cost", C.c_double), ("optimality", C.c_double),
        ("grad", C.c_double * JF_MAX_N), ("gram", C.c_double * (JF_MAX_N * JF_MAX_N)),
        ("pcov", C.c_double * (JF_MAX_N * JF_MAX_N)),
        ("status", C.c_int32), ("nfev", C.c_int32), ("njev", C.c_int32), ("nit", C.c_int32),
        ("n", C.c_int32), ("trace_len", C.c_int32),
        ("active_mask", C.c_int8 * JF_MAX_N),
        ("kernel_launches", C.c_int32), ("graph_reused", C.c_int32),
        ("t_upload_s", C.c_double), ("t_solve_s", C.c_double),
        ("t_epilogue_s", C.c_double), ("epilogue_cycles", C.c_double * 8),
        ("timeline_len", C.c_int32), ("pad2_", C.c_int32), ("timeline_ns", C.c_double * 64),
    ]


_lib = None


def load() -> C.CDLL:
    """Load libjfb200.so (built in-tree by build.py).  Raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2208_12187_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    dp = C.POINTER(C.c_double)
    ip = C.POINTER(C.c_int32)
    lib.jf_opts_default.argtypes = [C.POINTER(jf_opts)]
    lib.jf_opts_default.restype = None
    for f in ("jf_model_nparams", "jf_model_ydim", "jf_model_kslots"):
        getattr(lib, f).argtypes = [C.c_int32]
        getattr(lib, f).restype = C.c_int32
    lib.jf_curve_fit.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p,
                                 C.c_void_p, C.POINTER(jf_opts), C.POINTER(jf_result)]
    lib.jf_curve_fit.restype = C.c_int32
    lib.jf_curve_fit_batch.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                       C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(jf_opts), C.c_void_p]
    lib.jf_curve_fit_batch.restype = C.c_int32
    lib.jf_pass.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, dp, C.c_int32,
                            C.POINTER(jf_opts), dp, dp, dp, ip]
    lib.jf_pass.restype = C.c_int32
    lib.jf_residual_pass.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, dp, C.c_int32,
                                     C.POINTER(jf_opts), dp, ip]
    lib.jf_residual_pass.restype = C.c_int32
    lib.jf_pass_device.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                                   C.POINTER(jf_opts), C.c_int32, C.c_void_p]
    lib.jf_pass_device.restype = C.c_int32
    lib.jf_trust_region_step.argtypes = [dp, dp, C.c_int32, C.c_int64, C.c_double, C.c_double,
                                         C.POINTER(jf_opts), dp, dp, ip]
    lib.jf_trust_region_step.restype = C.c_int32
    lib.jf_select_step.argtypes = [dp, dp, dp, dp, dp, dp, dp, C.c_int32, C.c_double, C.c_double,
                                   C.POINTER(jf_opts), dp, dp, dp, ip]
    lib.jf_select_step.restype = C.c_int32
    lib.jf_comm_create.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
    lib.jf_comm_create.restype = C.c_int32
    lib.jf_comm_export.argtypes = [C.c_void_p, C.c_char_p]
    lib.jf_comm_export.restype = C.c_int32
    lib.jf_comm_connect.argtypes = [C.c_void_p, C.c_char_p]
    lib.jf_comm_connect.restype = C.c_int32
    lib.jf_comm_create_local.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
    lib.jf_comm_create_local.restype = C.c_int32
    lib.jf_comm_destroy.argtypes = [C.c_void_p]
    lib.jf_comm_destroy.restype = C.c_int32
    lib.jf_comm_set_timeout.argtypes = [C.c_void_p, C.c_int32]
    lib.jf_comm_set_timeout.restype = C.c_int32
    lib.jf_comm_bench.argtypes = [C.c_void_p, C.c_double, C.c_int32, dp, dp]
    lib.jf_comm_bench.restype = C.c_int32
    lib.jf_graph_cache_clear.argtypes = [C.c_int32]
    lib.jf_graph_cache_clear.restype = C.c_int32
    lib.jf_strerror.argtypes = [C.c_int32]
    lib.jf_strerror.restype = C.c_char_p
    lib.jf_version.argtypes = []
    lib.jf_version.restype = C.c_char_p
    _lib = lib
    return lib


EXPORTED = ["jf_opts_default", "jf_model_nparams", "jf_model_ydim", "jf_model_kslots", "jf_curve_fit",
            "jf_curve_fit_batch",
            "jf_pass", "jf_residual_pass", "jf_pass_device", "jf_trust_region_step", "jf_select_step",
            "jf_comm_create",
            "jf_comm_export", "jf_comm_connect", "jf_comm_create_local", "jf_comm_destroy",
            "jf_comm_set_timeout", "jf_comm_bench", "jf_graph_cache_clear", "jf_strerror", "jf_version"]
