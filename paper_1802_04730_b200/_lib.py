"""ctypes binding of libtcb.so (include/tcb.h). No fallback: importing this
module without the built library raises, and every call that fails raises
TcError carrying the reference's ErrorKind."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtcb.so")

TCB_F32, TCB_I32 = 0, 1
TCB_DEVICE, TCB_HOST = 0, 1
TCB_RUN_PROFILE, TCB_RUN_NOCHECK, TCB_RUN_ASYNC = 1, 2, 4
MATH_MODES = {"ffma": 0, "tf32": 1, "3xtf32": 3}

# ErrorKind order of proj/include/tc/support/diagnostics.h:36-68 (+2 additions)
ERROR_KINDS = [
    "Parse", "Name", "UnsupportedCall", "UnderConstrained", "Ambiguous", "EmptyRange",
    "LivenessInterference", "OutOfBounds", "UninitializedRead", "InvalidSchedule",
    "NoParallelOuterBand", "NotSinkable", "MappingInvalid", "PromotionBudget", "PromotionLogic",
    "IndexOutOfRange", "RaceDetected", "BarrierDivergence", "DegeneratePopulation",
    "NoViableCandidate", "CorruptStore", "MissingBinding", "ShapeMismatch", "Io", "Internal",
    "NoKernel", "Cuda",
]


class TcError(RuntimeError):
    """A failed tc-b200 call; ``kind`` is the reference ErrorKind name."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.kind = ERROR_KINDS[code - 1] if 0 < code <= len(ERROR_KINDS) else "Unknown"
        super().__init__(message)


class Tensor(C.Structure):
    _fields_ = [
        ("data", C.c_void_p),
        ("dtype", C.c_int32),
        ("rank", C.c_int32),
        ("shape", C.c_int64 * 8),
        ("location", C.c_int32),
        ("reserved", C.c_int32),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_1802_04730_b200/build.py` "
            "(tc-b200 has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    T = C.POINTER(Tensor)
    u64p = C.POINTER(C.c_uint64)
    sig = {
        "tcb_version": (C.c_char_p, []),
        "tcb_last_error": (C.c_char_p, []),
        "tcb_device_info": (C.c_int, [C.c_int, C.c_char_p, C.c_int]),
        "tcb_measure_peaks": (C.c_int, [C.c_int, C.c_char_p, C.c_int]),
        "tcb_engine_create": (C.c_int, [C.POINTER(C.c_void_p)]),
        "tcb_engine_destroy": (None, [C.c_void_p]),
        "tcb_builtin_ops": (C.c_char_p, []),
        "tcb_define": (C.c_int, [C.c_void_p, C.c_char_p]),
        "tcb_def_signature": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), C.c_char_p, C.c_int]),
        "tcb_infer_outputs": (C.c_int, [C.c_void_p, C.c_char_p, T, C.c_int, T, C.c_int]),
        "tcb_compile": (C.c_int, [C.c_void_p, C.c_char_p, T, C.c_int, T, C.c_int, C.c_char_p, u64p]),
        "tcb_compile_ex": (C.c_int, [C.c_void_p, C.c_char_p, T, C.c_int, T, C.c_int, C.c_char_p, C.c_int,
                                     u64p]),
        "tcb_run": (C.c_int, [C.c_void_p, C.c_uint64, T, C.c_int, T, C.c_int, C.c_void_p, C.c_int,
                              C.POINTER(C.c_int64)]),
        "tcb_check": (C.c_int, [C.c_void_p, C.c_uint64]),
        "tcb_release": (C.c_int, [C.c_void_p, C.c_uint64]),
        "tcb_shard_range": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "tcb_run_shard": (C.c_int, [C.c_void_p, C.c_uint64, T, C.c_int, T, C.c_int, C.c_int, C.c_int,
                                    C.c_void_p, C.c_int]),
        "tcb_describe": (C.c_int, [C.c_void_p, C.c_uint64, C.c_char_p, C.c_int]),
        "tcb_tune": (C.c_int, [C.c_void_p, C.c_char_p, T, C.c_int, T, C.c_int, C.c_char_p,
                               C.c_char_p, C.c_int]),
        "tcb_cache_load": (C.c_int, [C.c_char_p]),
        "tcb_cache_save": (C.c_int, [C.c_char_p]),
        "tcb_cache_size": (C.c_int, []),
        "tcb_cache_purge": (C.c_int, []),
        "tcb_cache_set_history": (C.c_int, [C.c_char_p]),
        "tcb_cache_serialize": (C.c_int, [C.c_char_p, C.c_int]),
        "tcb_cache_deserialize": (C.c_int, [C.c_char_p]),
        "tcb_cache_lookup": (C.c_int, [C.c_void_p, C.c_char_p, T, C.c_int, T, C.c_int,
                                       C.POINTER(C.c_int), C.c_char_p, C.c_int]),
        "tcb_cache_inject": (C.c_int, [C.c_void_p, C.c_char_p, T, C.c_int, T, C.c_int, C.c_char_p,
                                       C.c_int64]),
        "tcb_canonical": (C.c_int, [C.c_void_p, C.c_char_p, T, C.c_int, T, C.c_int, C.c_char_p,
                                    C.c_int, C.c_char_p, C.c_int]),
        "tcb_session_inputs": (C.c_int, [C.c_void_p, C.c_char_p, T, C.c_int, T, C.c_int,
                                         C.c_uint64]),
        "tcb_fill_uniform": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double,
                                       C.c_double]),
        "tcb_options_validate": (C.c_int, [C.c_char_p]),
        "tcb_options_normalize": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int]),
        "tcb_options_digest": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int]),
        "tcb_options_baseline": (C.c_int, [C.c_int, C.c_char_p, C.c_int]),
        "tcb_options_default": (C.c_int, [C.c_void_p, C.c_char_p, T, C.c_int, T, C.c_int,
                                          C.c_char_p, C.c_int]),
        "tcb_tensor_file_write": (C.c_int, [C.c_char_p, T]),
        "tcb_tensor_file_read": (C.c_int, [C.c_char_p, T]),
        "tcb_tensor_file_free": (None, [C.c_void_p]),
        "tcb_def_params": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int]),
        "tcb_cache_entries": (C.c_int, [C.c_char_p, C.c_int]),
        "tcb_concat_cols": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_int, C.c_int64,
                                      C.c_void_p, C.c_void_p]),
        "tcb_host_alloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_int64]),
        "tcb_host_free": (C.c_int, [C.c_void_p]),
        "tcb_device_alloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_int64]),
        "tcb_device_free": (C.c_int, [C.c_void_p]),
        "tcb_copy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
        "tcb_stream_sync": (C.c_int, [C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

# every symbol the C header declares (checked by tests/test_capi_symbols.py)
EXPORTED = [
    "tcb_version", "tcb_last_error", "tcb_device_info", "tcb_measure_peaks", "tcb_engine_create", "tcb_engine_destroy",
    "tcb_define", "tcb_builtin_ops", "tcb_def_signature", "tcb_infer_outputs", "tcb_compile",
    "tcb_compile_ex",
    "tcb_run", "tcb_shard_range", "tcb_run_shard", "tcb_release", "tcb_check", "tcb_describe", "tcb_tune", "tcb_cache_load", "tcb_cache_save",
    "tcb_cache_size", "tcb_cache_purge", "tcb_cache_set_history", "tcb_cache_serialize",
    "tcb_cache_deserialize", "tcb_cache_lookup", "tcb_cache_inject", "tcb_canonical",
    "tcb_session_inputs", "tcb_fill_uniform", "tcb_options_validate", "tcb_options_normalize",
    "tcb_options_digest", "tcb_options_baseline", "tcb_options_default", "tcb_host_alloc",
    "tcb_host_free", "tcb_device_alloc", "tcb_device_free", "tcb_copy", "tcb_stream_sync", "tcb_tensor_file_write", "tcb_tensor_file_read", "tcb_tensor_file_free", "tcb_def_params",
    "tcb_cache_entries", "tcb_concat_cols",
]


def check(rc: int):
    if rc != 0:
        raise TcError(rc, lib.tcb_last_error().decode())


def buf(n=1 << 16):
    return C.create_string_buffer(n)
