"""ctypes binding of libsr.so, the C-ABI kernel library (include/sr.h).

There is no CPU fallback: importing a compute entry without the built
library or without a CUDA device raises immediately.
"""
import ctypes
import os

from .errors import NonFiniteError, SeparationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SR_LIB_PATH") or os.path.join(_HERE, "libsr.so")  # override: A/B builds (tools/)

SR_OK, SR_EINVAL, SR_ESEPARATION, SR_ENONFINITE, SR_ECUDA = 0, 1, 2, 3, 4
SR_FLAG_SEPARATION, SR_FLAG_NONFINITE = 1, 2
SR_OP_N, SR_OP_C = 0, 1
SR_MAT_F64, SR_MAT_C64, SR_MAT_C128, SR_MAT_DD = 0, 1, 2, 3

_p = ctypes.c_void_p
_i = ctypes.c_int
_ll = ctypes.c_longlong
_d = ctypes.c_double
_f = ctypes.c_float
_sz = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/sr.h one to one
SIGNATURES = {
    "sr_version": (_i, []),
    "sr_last_error": (ctypes.c_char_p, []),
    "sr_kernel_launches": (ctypes.c_ulonglong, []),
    "sr_zgemm_f64": (_i, [_i, _i, _i, _i, _d, _d, _p, _p, _ll, _p, _p, _ll, _p, _p, _ll, _p]),
    "sr_cgemm_c64": (_i, [_i, _i, _i, _i, _p, _ll, _p, _ll, _p, _ll, _p]),
    "sr_split_lp_c64": (_i, [_i, _p, _p, _ll, _p, _p, _ll, _p, _p, _sz, _p]),
    "sr_fro_norm_f64": (_i, [_i, _i, _p, _p, _ll, _p, _p, _sz, _p]),
    "sr_striu_norm_f64": (_i, [_i, _p, _p, _ll, _p, _p, _sz, _p]),
    "sr_diag_correction_c64": (_i, [_i, _p, _p, _ll, _p, _f, _p, _p, _p]),
    "sr_diag_correction_c128": (_i, [_i, _p, _p, _ll, _p, _d, _p, _p, _p]),
    "sr_downcast_c64": (_i, [_i, _i, _p, _p, _ll, _p, _ll, _p]),
    "sr_trisolve_workspace_bytes": (_sz, [_i, _i]),
    "sr_trisolve_c64": (_i, [_i, _p, _p, _ll, _p, _f, _p, _p, _p, _sz, _p]),
    "sr_trisolve_c128": (_i, [_i, _p, _p, _ll, _p, _d, _p, _p, _p, _sz, _p]),
    "sr_skew_c64": (_i, [_i, _p, _ll, _p, _p, _p, _p, _sz, _p]),
    "sr_sigma_merged_f64": (_i, [_i, _i, _p, _p, _p, _ll, _p, _p, _p, _p, _p, _ll, _p, _p, _ll, _i, _p]),
    "sr_fused_lp_operand_c64": (_i, [_i, _p, _p, _ll, _p, _p, _ll, _p, _p]),
    "sr_sigma_ns_f64": (_i, [_i, _p, _p, _ll, _p, _p, _ll, _p]),
    "sr_triu_inplace_f64": (_i, [_i, _p, _p, _ll, _p]),
    "sr_reduce_workspace_bytes": (_sz, []),
    "sr_split_lp_c128": (_i, [_i, _p, _p, _ll, _p, _p, _ll, _p, _p, _sz, _p]),
    "sr_skew_c128": (_i, [_i, _p, _ll, _p, _p, _p, _p, _sz, _p]),
    "sr_pack_c128": (_i, [_i, _i, _p, _p, _ll, _p, _ll, _p]),
    "sr_sigma_merged_dd": (_i, [_i, _p, _p, _p, _p, _p, _ll, _p, _p, _p, _p, _p, _ll, _p, _p, _p, _p, _ll, _i, _p]),
    "sr_oz_exponents": (_i, [_i, _i, _i, _p, _p, _ll, _i, _p, _p]),
    "sr_oz_exponents_bound": (_i, [_i, _i, _i, _p, _p, _ll, _i, _p, _p, _p, _p, _p]),
    "sr_oz_encode": (_i, [_i, _i, _i, _p, _p, _p, _p, _ll, _i, _i, _i, _p, _i, _i, _p, _p, _ll, _p]),
    "sr_oz_encode_dual": (_i, [_i, _i, _i, _p, _p, _p, _p, _ll, _p, _i, _i, _p, _p, _p, _ll, _p]),
    "sr_oz_gemm_i8": (_i, [_i, _i, _i, _i, _p, _p, _i, _ll, _p, _i, _ll, _p, _ll, _i, _i, _p]),
    "sr_oz_decode": (_i, [_i, _i, _i, _i, _p, _p, _ll, _p, _i, _p, _i, _d, _d, _i, _p, _p, _p, _p, _ll, _d, _i,
                          _p, _p, _p, _p, _ll, _i, _i, _p]),
    "sr_oz_gemm_i8_gauss": (_i, [_i, _i, _i, _i, _p, _p, _i, _ll, _p, _i, _ll, _p, _ll, _i, _i, _p]),
    "sr_oz_decode_gauss": (_i, [_i, _i, _i, _i, _p, _p, _ll, _p, _i, _p, _i, _d, _d, _i, _p, _p, _ll, _d, _i,
                                _p, _p, _ll, _i, _i, _p]),
    "sr_oz_config": (_i, [_i, _i]),
    "sr_dd_add": (_i, [_i, _i, _p, _p, _ll, _p, _p, _ll, _i, _p, _p, _ll, _p]),
    "sr_dd_scale": (_i, [_i, _i, _p, _p, _ll, _d, _p, _p, _ll, _p]),
    "sr_stril_split_f64": (_i, [_i, _i, _p, _ll, _p, _ll, _p, _ll, _p]),
    "sr_fro_norm_dd_workspace_bytes": (_sz, [_ll]),
    "sr_fro_norm_dd": (_i, [_i, _i, _p, _p, _p, _p, _ll, _p, _p, _sz, _p]),
    "sr_zgemm_dd_fma": (_i, [_i, _i, _i, _i, _p, _p, _p, _p, _ll, _p, _p, _p, _p, _ll, _p, _p, _p, _p, _ll, _p]),
    "sr_power_norm_workspace_bytes": (_sz, [_i]),
    "sr_power_norm_c64": (_i, [_i, _p, _ll, _i, _i, _d, _p, _sz, _p]),
    "sr_finite_flag_f64": (_i, [_i, _i, _p, _p, _ll, _p, _i, _p]),
    "sr_phase_perm_workspace_bytes": (_sz, [_i]),
    "sr_phase_perm_scan_f64": (_i, [_i, _p, _p, _ll, _p, _p, _p, _sz, _p]),
    "sr_split_lp_block_c64": (_i, [_i, _i, _i, _p, _p, _ll, _p, _p, _ll, _p, _p, _sz, _p]),
    "sr_fused_lp_operand_block_c64": (_i, [_i, _i, _p, _p, _ll, _p, _p, _ll, _p, _p]),
}

_lib = None


def load():
    """Load libsr.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libsr.so not built (run __graft_entry__.build() or make -C %s)" % _HERE)
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc, what):
    if rc == SR_OK:
        return
    msg = "%s failed (status %d)" % (what, rc)
    err = load().sr_last_error()
    if err:
        msg += ": " + err.decode(errors="replace")
    if rc == SR_ESEPARATION:
        raise SeparationError(msg)
    if rc == SR_ENONFINITE:
        raise NonFiniteError(msg)
    if rc == SR_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def call(name, *args):
    check(getattr(load(), name)(*args), name)
