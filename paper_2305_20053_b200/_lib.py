"""ctypes binding of libsaadino.so (the C ABI in include/saadino.h).

The library is mapped on first use (the first call through `lib`), not at
import: the package's host-side modules (workloads, fileio, the reference-
facing API types) import without the CUDA engine, so e.g. bench.py's CPU
reference arm never maps it.  The product path has no CPU fallback: the
first engine call raises ImportError, naming the build command, when the
shared library is missing.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SDN_LIB_VARIANT=name loads libsaadino_<name>.so (build-variant A/B studies)
LIB_PATH = os.path.join(_HERE, "libsaadino" + (("_" + os.environ["SDN_LIB_VARIANT"]) if os.environ.get("SDN_LIB_VARIANT") else "") + ".so")

SDN_OK = 0
ACT = {"identity": 0, "tanh": 1, "softplus": 2, "sigmoid": 3, "elu": 4, "softmax": 5}
RISK = {"mean": 0, "cvar": 1, "meanvar": 2, "cvar_exact": 3}
QOI = {"reduced": 0, "decoded": 1}
GEMM = {"auto": 0, "simt": 1, "tc": 2}
STATS_LEN = 8
PROF_CLASSES = ["fwd_gemm", "bwd_gemm", "qoi", "select", "compact", "seed", "colsum", "finalize", "zbias",
                "other", "refine", "tangent_gemm", "decode_gemm"]


class Config(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("widths", C.POINTER(C.c_int32)), ("r_m", C.c_int32),
                ("d_z", C.c_int32), ("activation", C.c_int32), ("residual", C.c_int32),
                ("gemm", C.c_int32), ("device", C.c_int32), ("max_samples", C.c_int64)]


class Risk(C.Structure):
    _fields_ = [("kind", C.c_int32), ("qoi", C.c_int32), ("beta", C.c_double), ("eps", C.c_double),
                ("t", C.c_double), ("alpha", C.c_double), ("need_grad", C.c_int32)]


class Result(C.Structure):
    _fields_ = [("value", C.c_double), ("grad_t", C.c_double), ("n_samples", C.c_int64),
                ("n_selected", C.c_int64), ("q_mean", C.c_double), ("q_var", C.c_double),
                ("n_refined", C.c_int64)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_I64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes); kept in sync with include/saadino.h
SIGNATURES = {
    "sdn_last_error": (C.c_char_p, []),
    "sdn_version": (C.c_int, []),
    "sdn_create": (C.c_int, [C.POINTER(Config), C.POINTER(_P)]),
    "sdn_destroy": (C.c_int, [_P]),
    "sdn_set_stream": (C.c_int, [_P, _P]),
    "sdn_synchronize": (C.c_int, [_P]),
    "sdn_set_model": (C.c_int, [_P, C.POINTER(_F), C.POINTER(_F), _F, _F, _F, _F]),
    "sdn_set_tracking": (C.c_int, [_P, _F, C.c_double]),
    "sdn_set_decoder": (C.c_int, [_P, C.c_int64, _F, _F, _F, _F]),
    "sdn_set_decoder_csr": (C.c_int, [_P, C.c_int64, _F, _F, C.POINTER(C.c_int64), C.POINTER(C.c_int32), _F, _F]),
    "sdn_set_samples": (C.c_int, [_P, _P, C.c_int64, C.c_int64, C.c_int32]),
    "sdn_encode_fields": (C.c_int, [_P, _P, C.c_int64, C.c_int64, _F, _F, C.c_float, C.c_int64, C.c_int32]),
    "sdn_eval": (C.c_int, [_P, _D, C.POINTER(Risk), C.POINTER(Result), _D, _I64]),
    "sdn_eval_multi": (C.c_int, [_P, _D, C.POINTER(Risk), C.c_int32, C.POINTER(Result), _D, _I64]),
    "sdn_eval_multi_launch": (C.c_int, [_P, _D, C.POINTER(Risk), C.c_int32, C.c_int32]),
    "sdn_eval_multi_wait": (C.c_int, [_P, C.POINTER(Result), _D, _I64]),
    "sdn_eval_samples": (C.c_int, [_P, _D, C.c_int32, _D, _D]),
    "sdn_forward_batch": (C.c_int, [_P, _F, _F, C.c_int64, _F]),
    "sdn_jacobian_batch": (C.c_int, [_P, _F, _F, C.c_int64, C.c_int32, _F]),
    "sdn_jacobian_samples": (C.c_int, [_P, _D, C.c_int32, _P]),
    "sdn_lift": (C.c_int, [_P, _F, C.c_int64, _F]),
    "sdn_select_topk": (C.c_int, [_P, _P, C.c_int64, C.c_int64, C.c_int32, _I64]),
    "sdn_partial_len": (C.c_int, [_P]),
    "sdn_eval_forward": (C.c_int, [_P, _D, C.POINTER(Risk), _P]),
    "sdn_eval_candidates": (C.c_int, [_P, C.c_int64, _P]),
    "sdn_eval_select": (C.c_int, [_P, _P, C.c_int32, C.c_int64]),
    "sdn_eval_refine_band": (C.c_int, [_P]),
    "sdn_eval_keep_selection": (C.c_int, [_P, C.c_int32]),
    "sdn_eval_selection": (C.c_int, [_P, C.c_int32, C.c_int64, _I64]),
    "sdn_train_setup": (C.c_int, [_P, _F, _F, _F, _F, C.c_int64, C.c_int32]),
    "sdn_train_set_params": (C.c_int, [_P, C.POINTER(_D), C.POINTER(_D), _D, _D, _D]),
    "sdn_train_set_mask": (C.c_int, [_P, C.POINTER(_D), C.POINTER(_D)]),
    "sdn_train_get_params": (C.c_int, [_P, C.POINTER(_D), C.POINTER(_D)]),
    "sdn_train_get_grad": (C.c_int, [_P, C.POINTER(_D), C.POINTER(_D)]),
    "sdn_train_step": (C.c_int, [_P, _I64, C.c_int32, C.c_double, C.c_double, C.c_int64, _D]),
    "sdn_eval_backward_multi": (C.c_int, [_P, C.POINTER(Risk), C.c_int32, _P, _P]),
    "sdn_eval_backward": (C.c_int, [_P, _P, _P]),
    "sdn_eval_set_risk": (C.c_int, [_P, C.POINTER(Risk)]),
    "sdn_eval_finish": (C.c_int, [_P, _P, _P, C.POINTER(Result), _D]),
    "sdn_last_q": (C.c_int, [_P, C.POINTER(_P), _I64]),
    "sdn_last_qsel": (C.c_int, [_P, C.POINTER(_P), _I64]),
    "sdn_kernel_launches": (C.c_int64, [_P]),
    "sdn_profile": (C.c_int, [_P, C.c_int32]),
    "sdn_debug_gemm": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, _D]),
    "sdn_profile_read": (C.c_int, [_P, C.c_int32, _D, _D, _D, _I64]),
    "sdn_last_device_ms": (C.c_int, [_P, _D]),
}


class SaadinoError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the SAA engine has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class _LazyLib:
    """Proxy that CDLLs libsaadino.so on first attribute access."""

    _lib = None

    def __getattr__(self, name):
        if _LazyLib._lib is None:
            _LazyLib._lib = _load()
        return getattr(_LazyLib._lib, name)

    @staticmethod
    def loaded() -> bool:
        return _LazyLib._lib is not None


lib = _LazyLib()


def check(rc: int, what: str = ""):
    if rc != SDN_OK:
        msg = lib.sdn_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise SaadinoError(f"{what} failed ({rc}): {msg}")


def fptr(a):
    return a.ctypes.data_as(_F)


def dptr(a):
    return a.ctypes.data_as(_D)


def i64ptr(a):
    return a.ctypes.data_as(_I64)
