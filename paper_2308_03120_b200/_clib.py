"""ctypes binding of libb200mat.so (include/b200mat.h).

This is the only module that touches the native library.  There is no
fallback: if the shared object is missing or a call fails, an exception is
raised.  The structures below are field-for-field images of the C structs.
"""
from __future__ import annotations

import ctypes
import os
import pathlib

from .errors import BufferError_, DevmatError

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = _HERE / "libb200mat.so"

# ---- constants (include/b200mat.h) -------------------------------------------------
BM_OK, BM_ERR_CUDA, BM_ERR_ARG, BM_ERR_NOTIMPL, BM_ERR_EMPTY, BM_ERR_JIT, BM_ERR_NODEVICE, BM_ERR_PEER = range(8)
BM_F32, BM_F64, BM_I32, BM_U64 = range(4)
DTYPE_CODE = {"f32": BM_F32, "f64": BM_F64, "i32": BM_I32, "u64": BM_U64}

(BM_K_EWISE, BM_K_REDUCE, BM_K_RDIM, BM_K_GEMM, BM_K_COPY, BM_K_TRANSPOSE, BM_K_FILL, BM_K_EYE,
 BM_K_LINSPACE, BM_K_RANDU, BM_K_RANDN, BM_K_STRIDED_COPY, BM_K_LOGISTIC_GRAD, BM_K_PRED_COUNT,
 BM_K_PRED_FIND, BM_K_GEMM_FUSED, BM_K_RDIM_FUSED, BM_K_GEMM_EPI) = range(1, 19)
BM_CMP_GT, BM_CMP_LT, BM_CMP_GE, BM_CMP_LE, BM_CMP_EQ, BM_CMP_NE = range(6)
PRED_CODE = {">": BM_CMP_GT, "<": BM_CMP_LT, ">=": BM_CMP_GE, "<=": BM_CMP_LE, "==": BM_CMP_EQ, "!=": BM_CMP_NE}

BM_P_LOAD, BM_P_UNARY, BM_P_SCALAR, BM_P_GLUE = range(4)
UNARY_CODE = {"eop_exp": 0, "eop_log": 1, "eop_log10": 2, "eop_sqrt": 3, "eop_square": 4, "eop_pow": 5,
              "eop_abs": 6, "eop_cos": 7, "eop_sin": 8, "eop_tan": 9, "eop_acos": 10, "eop_asin": 11,
              "eop_atan": 12}
SCALAR_CODE = {"eop_scalar_plus": 0, "eop_scalar_minus_pre": 1, "eop_scalar_minus_post": 2,
               "eop_scalar_times": 3, "eop_scalar_div_pre": 4, "eop_scalar_div_post": 5}
GLUE_CODE = {"eglue_plus": 0, "eglue_minus": 1, "eglue_schur": 2, "eglue_div": 3}
BM_R_NONE, BM_R_ACCU, BM_R_MIN, BM_R_MAX, BM_R_DOT, BM_R_MEAN, BM_R_VAR = range(7)
(BM_MOV_EXTRACT, BM_MOV_INSERT, BM_MOV_RESIZE, BM_MOV_RESHAPE, BM_MOV_JOIN_ROWS, BM_MOV_JOIN_COLS,
 BM_MOV_DIAGMAT, BM_MOV_DIAGVEC, BM_MOV_REPMAT) = range(9)

BM_MAX_INPUTS = 16
BM_MAX_SCALARS = 16
BM_MAX_PROG = 64


class View(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("offset", ctypes.c_int64), ("count", ctypes.c_int64),
                ("stride", ctypes.c_int64), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("lda", ctypes.c_int64), ("dtype", ctypes.c_int32), ("is_block", ctypes.c_int32)]


class Invocation(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_inputs", ctypes.c_int32),
                ("inputs", View * BM_MAX_INPUTS), ("has_output", ctypes.c_int32), ("output", View),
                ("n_scalars", ctypes.c_int32), ("fscalars", ctypes.c_double * BM_MAX_SCALARS),
                ("iscalars", ctypes.c_int64 * BM_MAX_SCALARS), ("n_prog", ctypes.c_int32),
                ("prog", ctypes.c_int32 * (3 * BM_MAX_PROG)), ("compute_dtype", ctypes.c_int32),
                ("reduce_op", ctypes.c_int32), ("dim", ctypes.c_int32), ("trans_a", ctypes.c_int32),
                ("trans_b", ctypes.c_int32), ("sub_kind", ctypes.c_int32), ("iparams", ctypes.c_int64 * 8)]


class Counters(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("jit_compiles", ctypes.c_int64),
                ("jit_cache_hits", ctypes.c_int64), ("bytes_h2d", ctypes.c_int64), ("bytes_d2h", ctypes.c_int64)]


# every symbol include/b200mat.h declares, with its ctypes signature
_VP, _I32, _I64, _CP = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_char_p
SIGNATURES = {
    "bm_abi_version": ([], ctypes.c_int),
    "bm_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "bm_init": ([ctypes.c_int], ctypes.c_int),
    "bm_shutdown": ([], ctypes.c_int),
    "bm_device_info": ([ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                        ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "bm_set_stream": ([_VP], ctypes.c_int),
    "bm_get_stream": ([], _VP),
    "bm_last_error": ([], _CP),
    "bm_alloc": ([_I64, ctypes.POINTER(_VP)], ctypes.c_int),
    "bm_free": ([_VP], ctypes.c_int),
    "bm_free_async": ([_VP], ctypes.c_int),
    "bm_h2d": ([_VP, _VP, _I64], ctypes.c_int),
    "bm_d2h": ([_VP, _VP, _I64], ctypes.c_int),
    "bm_d2d": ([_VP, _VP, _I64], ctypes.c_int),
    "bm_h2d_async": ([_VP, _VP, _I64], ctypes.c_int),
    "bm_d2h_async": ([_VP, _VP, _I64], ctypes.c_int),
    "bm_read_elems": ([_VP, _I32, ctypes.POINTER(_I64), _I64, _VP], ctypes.c_int),
    "bm_write_elem": ([_VP, _I32, _I64, _VP], ctypes.c_int),
    "bm_host_alloc_pinned": ([_I64, ctypes.POINTER(_VP)], ctypes.c_int),
    "bm_host_free_pinned": ([_VP], ctypes.c_int),
    "bm_enqueue": ([ctypes.POINTER(Invocation)], ctypes.c_int),
    "bm_execute_reduce": ([ctypes.POINTER(Invocation), _VP], ctypes.c_int),
    "bm_reduce_to_device": ([ctypes.POINTER(Invocation), _VP], ctypes.c_int),
    "bm_combine_partials": ([_VP, _I64, _I32, _I32, _VP], ctypes.c_int),
    "bm_combine_partials_to_device": ([_VP, _I64, _I32, _I32, _VP], ctypes.c_int),
    "bm_exchange_alloc": ([_I32, ctypes.POINTER(_VP), _VP], ctypes.c_int),
    "bm_exchange_open": ([_VP, ctypes.POINTER(_VP)], ctypes.c_int),
    "bm_exchange_alloc_vec": ([_I32, _I64, ctypes.POINTER(_VP), _VP], ctypes.c_int),
    "bm_exchange_gsum": ([_VP, _I64, _VP, ctypes.POINTER(_VP), _I32, _I32, ctypes.c_uint64, _I64, _VP, _VP],
                         ctypes.c_int),
    "bm_exchange_rows": ([_VP, _I64, _I32, _I32, ctypes.POINTER(_VP), _I32, _I32, ctypes.c_uint64, _I64, _VP],
                         ctypes.c_int),
    "bm_exchange_close": ([_VP, _I32], ctypes.c_int),
    "bm_reduce_to_device_exchange": ([ctypes.POINTER(Invocation), _VP, _VP, _I32, _I32, ctypes.c_uint64], ctypes.c_int),
    "bm_exchange_combine": ([_VP, ctypes.POINTER(_VP), _I32, _I32, ctypes.c_uint64, _I32, _I32, _VP], ctypes.c_int),
    "bm_sync": ([], ctypes.c_int),
    "bm_poll_device_error": ([], ctypes.c_int),
    "bm_stream_busy": ([], ctypes.c_int),
    "bm_get_counters": ([ctypes.POINTER(Counters)], ctypes.c_int),
    "bm_set_cache_dir": ([_CP], ctypes.c_int),
    "bm_jit_compile_only": ([ctypes.POINTER(Invocation)], ctypes.c_int),
    "bm_gemm": ([_I32, _I32, _I32, _I64, _I64, _I64, _VP, _I64, _VP, _I64, _VP, _I64], ctypes.c_int),
    "bm_set_gemm_algo": ([_I32], ctypes.c_int),
}

_lib = None


class DeviceError(DevmatError, RuntimeError):
    """A CUDA / NVRTC failure inside libb200mat.so."""


class PeerTimeoutError(DeviceError):
    """A cross-GPU exchange gave up waiting for a peer rank (BM_ERR_PEER): the
    sharded result is invalid.  Raised at the next synchronisation point."""


def lib() -> ctypes.CDLL:
    """Load libb200mat.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -m paper_2308_03120_b200.build or __graft_entry__.build()); "
            "there is no CPU fallback")
    h = ctypes.CDLL(str(LIB_PATH))
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(h, name)
        fn.argtypes = args
        fn.restype = res
    cache = os.environ.get("BM_CACHE_DIR")
    if cache is None:
        cache = str(_HERE / ".jitcache")
    if cache:
        os.makedirs(cache, exist_ok=True)
        h.bm_set_cache_dir(cache.encode())
    _lib = h
    return h


def last_error() -> str:
    msg = lib().bm_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a status code to the reference's exception types (errors.py)."""
    if rc == BM_OK:
        return
    msg = last_error()
    text = f"{what}: {msg}" if what else msg
    if rc == BM_ERR_EMPTY:
        raise ValueError(text)
    if rc == BM_ERR_NOTIMPL:
        raise NotImplementedError(text)
    if rc == BM_ERR_ARG:
        raise BufferError_(text)
    if rc == BM_ERR_PEER:
        raise PeerTimeoutError(text)
    raise DeviceError(text)
