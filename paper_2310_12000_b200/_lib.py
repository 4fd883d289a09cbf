"""ctypes binding of the in-tree CUDA library libvlgpx.so (include/vlgpx.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
compute entry point raises DeviceError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import STATUS, DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VLGPX_LIB") or os.path.join(_HERE, "libvlgpx.so")

_lock = threading.Lock()
_lib = None

c_int, c_int64, c_double, c_void_p = C.c_int, C.c_int64, C.c_double, C.c_void_p
P_int32 = C.POINTER(C.c_int32)
P_int64 = C.POINTER(C.c_int64)
P_double = C.POINTER(C.c_double)

# name -> (argtypes); every function returns int status unless listed in _RET
_SIGS = {
    "vl_version": [],
    "vl_last_error": [],
    "vl_ctx_create": [c_int, c_void_p, C.POINTER(c_void_p)],
    "vl_ctx_destroy": [c_void_p],
    "vl_ctx_sync": [c_void_p],
    "vl_ctx_info": [c_void_p, P_int64],
    "vl_knn_previous": [c_void_p, c_int64, c_int, c_int, c_void_p, c_int],
    "vl_knn_previous_dev": [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p],
    "vl_knn_query": [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p],
    "vl_pattern_create": [c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p, c_int, C.POINTER(c_void_p)],
    "vl_pattern_destroy": [c_void_p],
    "vl_pattern_perm": [c_void_p, c_void_p],
    "vl_pattern_info": [c_void_p, P_int64],
    "vl_pattern_solve_order": [c_void_p, c_int, P_int64, c_void_p],
    "vl_factor_build": [c_void_p, c_void_p, c_double, c_double, c_double, c_int, C.POINTER(c_void_p)],
    "vl_factor_destroy": [c_void_p],
    "vl_factor_get": [c_void_p, c_void_p, c_int, c_void_p],
    "vl_factor_set": [c_void_p, c_void_p, c_int, c_void_p],
    "vl_spmm": [c_void_p, c_void_p, c_int, c_int64, c_void_p, c_void_p],
    "vl_sptrsv": [c_void_p, c_void_p, c_int, c_int64, c_void_p, c_void_p],
}
class VlLik(C.Structure):
    _fields_ = [("family", C.c_int), ("shape", C.c_double)]


class VlNewtonCfg(C.Structure):
    _fields_ = [("mode_cg_tol", C.c_double), ("cg_max_iter", C.c_int), ("newton_max_iter", C.c_int),
                ("newton_grad_tol", C.c_double), ("newton_obj_tol", C.c_double), ("precond", C.c_int)]


_V = c_void_p
_SIGS.update({
    "vl_find_mode": [_V, _V, C.POINTER(VlLik), C.POINTER(VlNewtonCfg), _V, _V, _V, _V, _V, _V, _V, _V, c_int],
    "vl_probes_vadu": [_V, _V, _V, c_int64, _V, _V, _V, _V],
    "vl_pcg_vadu": [_V, _V, _V, c_int64, _V, _V, c_double, c_int, c_int, _V, _V, _V, _V, _V, c_int],
    "vl_factor_sums": [_V, _V, _V, _V],
    "vl_grad_probe_pass": [_V, _V, _V, _V, _V, _V, c_int64, _V, _V, _V, _V, c_int],
    "vl_precond_dinv": [_V, _V, c_int, _V, _V],
    "vl_pcg_eq6": [_V, _V, _V, _V, c_int, c_int64, _V, _V, c_double, c_int, c_int, _V, _V, _V, _V, _V, c_int],
    "vl_probes_eq6": [_V, _V, _V, c_int, c_int64, _V, _V, _V, _V],
    "vl_sum_log": [_V, c_int64, _V, _V],
    "vl_grad_scalar_terms": [_V, _V, _V, _V, _V],
    "vl_grad_dbeta": [_V, c_int64, _V, _V, _V, _V, _V, c_int64, _V],
    "vl_gamma_xi_terms": [_V, _V, _V, _V, _V, _V, _V, _V, _V],
})
_RET = {"vl_last_error": C.c_char_p}

# functions declared in include/vlgpx.h (tests check the export table)
EXPORTED = sorted(_SIGS)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"native library {LIB_PATH} is missing; run `python -m paper_2310_12000_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RET.get(name, c_int)
        _lib = L
    return _lib


def check(status):
    if status != 0:
        msg = lib().vl_last_error()
        msg = msg.decode() if msg else f"status {status}"
        raise STATUS.get(status, DeviceError)(msg)


def call(name, *args):
    check(getattr(lib(), name)(*args))


def ptr(a):
    """Raw pointer of a numpy array or torch tensor (contiguity checked)."""
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(a.data_ptr())
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(c_void_p)

_SIGS.update({
    "vl_prof_enable": [c_void_p, c_int],
    "vl_prof_reset": [c_void_p],
    "vl_prof_only": [c_void_p, C.c_char_p],
    "vl_prof_report": [c_void_p, C.c_char_p, c_int, P_int64],
})
EXPORTED = sorted(_SIGS)

_SIGS.update({
    "vl_grad_probe_pass_split": [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                 c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int],
})
EXPORTED = sorted(_SIGS)

_SIGS.update({
    "vl_lrac_create": [c_void_p, c_void_p, c_int, c_double, C.POINTER(c_void_p), c_void_p, C.POINTER(c_int)],
    "vl_lrac_destroy": [c_void_p],
    "vl_lrac_get_L": [c_void_p, c_void_p, c_void_p],
    "vl_lrac_prepare": [c_void_p, c_void_p, c_void_p, C.POINTER(c_void_p), c_void_p],
    "vl_lracw_destroy": [c_void_p],
    "vl_lrac_apply_inv": [c_void_p, c_void_p, c_int64, c_void_p, c_void_p],
    "vl_lrac_pcg": [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_double, c_int, c_int, c_void_p, c_void_p,
                    c_void_p, c_void_p, c_void_p, c_int],
    "vl_lrac_solve_system": [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_double, c_int, c_void_p],
    "vl_apply_sigma_tilde": [c_void_p, c_void_p, c_int64, c_void_p, c_void_p],
    "vl_lrac_probes": [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "vl_lrac_grad": [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                     c_void_p, c_void_p, c_void_p, c_int],
    "vl_probes_rademacher": [c_void_p, c_void_p, c_int64, c_int64, c_int64, C.c_uint64, c_void_p],
    "vl_probes_given": [c_void_p, c_void_p, c_void_p, c_int, c_int64, c_void_p, c_void_p, c_void_p],
    "vl_dgemm": [c_void_p, c_int, c_int, c_int64, c_int64, c_int64, c_double, c_void_p, c_int64, c_void_p, c_int64,
                 c_double, c_void_p, c_int64, c_void_p, c_int],
    "vl_dtrtri_lower": [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64],
    "vl_lrac_grad_split": [c_void_p, c_void_p, c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                           c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int],
    "vl_lowrank_create": [c_void_p, c_void_p, c_int, c_int, c_double, c_void_p, c_void_p, c_void_p],
    "vl_lowrank_einv": [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_void_p],
    "vl_lowrank_prepare": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p],
    "vl_diag_sigma_tilde": [c_void_p, c_void_p, c_void_p],
    "vl_find_mode_lowrank": [c_void_p, c_void_p, c_void_p, c_int, c_void_p, C.POINTER(VlLik), C.POINTER(VlNewtonCfg),
                             c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int],
    "vl_pred_create": [c_void_p, c_void_p, c_double, c_double, c_double, c_void_p, c_int64, c_void_p, c_int,
                       c_void_p],
    "vl_pred_destroy": [c_void_p],
    "vl_pred_get": [c_void_p, c_void_p, c_int, c_void_p],
    "vl_pred_mean": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "vl_pred_z3": [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p],
    "vl_pred_accum": [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p],
    "vl_pred_lanczos": [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int64, c_void_p, c_void_p, c_double,
                        c_void_p, c_void_p],
    "vl_find_mode_lrac": [c_void_p, c_void_p, c_void_p, C.POINTER(VlLik), C.POINTER(VlNewtonCfg), c_void_p, c_void_p,
                          c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int],
})
EXPORTED = sorted(_SIGS)
