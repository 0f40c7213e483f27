"""ctypes binding of the C ABI (include/shampoo_b200.h) -> libshampoo_b200.so.

The library is built in-tree (``python -m paper_2309_06497_b200.build_native``).
There is no fallback: if the .so is missing, importing the optimizer raises.
"""

from __future__ import annotations

import ctypes as C
import os

from .config import NativeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libshampoo_b200.so")

OK = 0
ERR_INVALID_ARGUMENT = -1
ERR_INVALID_GROUP = -2
ERR_NONFINITE_GRAD = -3
ERR_CUDA = -4
ERR_OUT_OF_MEMORY = -5
ERR_SHAPE = -6
ERR_UNSUPPORTED = -7

DTYPE_F32 = 0
DTYPE_F64 = 1
MAX_ORDER = 8

BLOCK_SHAMPOO, BLOCK_GRAFT_ONLY, BLOCK_ADAGRAD, BLOCK_DIAGONAL = 0, 1, 2, 3
KIND_NAMES = {BLOCK_SHAMPOO: "shampoo", BLOCK_GRAFT_ONLY: "graft_only",
              BLOCK_ADAGRAD: "adagrad", BLOCK_DIAGONAL: "diagonal"}


class BlockInfo(C.Structure):
    _fields_ = [
        ("block_id", C.c_int32), ("param_index", C.c_int32), ("block_index", C.c_int32),
        ("order", C.c_int32), ("owner_rank", C.c_int32), ("kind", C.c_int32),
        ("var_count", C.c_int64), ("gather_offset", C.c_int64),
        ("lo", C.c_int64 * MAX_ORDER), ("hi", C.c_int64 * MAX_ORDER),
    ]


class Config(C.Structure):
    _fields_ = [
        ("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("epsilon", C.c_double),
        ("momentum", C.c_double), ("use_nesterov", C.c_int32), ("weight_decay", C.c_double),
        ("use_decoupled_weight_decay", C.c_int32), ("use_bias_correction", C.c_int32),
        ("max_preconditioner_dim", C.c_int64), ("precondition_frequency", C.c_int64),
        ("start_preconditioning_step", C.c_double), ("exponent_override", C.c_int32),
        ("exponent_multiplier", C.c_double), ("grafting", C.c_int32),
        ("grafting_epsilon", C.c_double), ("grafting_beta2", C.c_double),
        ("large_dim_method", C.c_int32), ("solver", C.c_int32), ("newton_tolerance", C.c_double),
        ("precision", C.c_int32), ("gather_dtype", C.c_int32),
    ]


class GuardStatsC(C.Structure):
    _fields_ = [("primary", C.c_int64), ("double_retry", C.c_int64),
                ("fallback_previous", C.c_int64), ("fallback_identity", C.c_int64)]


_P = C.c_void_p
_I32, _I64, _D = C.c_int32, C.c_int64, C.c_double
_PI32, _PI64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)

# name -> (restype, argtypes); mirrors include/shampoo_b200.h exactly
SIGNATURES = {
    "shampoo_last_error": (C.c_char_p, []),
    "shampoo_version": (C.c_char_p, []),
    "shampoo_merge_dims": (C.c_int, [_PI64, _I32, _I64, _PI64, _PI32]),
    "shampoo_plan_create": (C.c_int, [_PI64, _PI32, _I32, _I64, _I32, _I32, _I32, C.POINTER(_P)]),
    "shampoo_plan_destroy": (None, [_P]),
    "shampoo_plan_num_blocks": (_I32, [_P]),
    "shampoo_plan_num_params": (_I32, [_P]),
    "shampoo_plan_block": (C.c_int, [_P, _I32, C.POINTER(BlockInfo)]),
    "shampoo_plan_param": (C.c_int, [_P, _I32, _PI64, _PI32, _PI32]),
    "shampoo_plan_counters": (C.c_int, [_P, _PI64]),
    "shampoo_plan_max_payload": (_I64, [_P]),
    "shampoo_plan_group_size": (_I32, [_P]),
    "shampoo_plan_world_size": (_I32, [_P]),
    "shampoo_ctx_create": (C.c_int, [_P, C.POINTER(Config), _I32, _I32, C.POINTER(_P)]),
    "shampoo_ctx_destroy": (None, [_P]),
    "shampoo_ctx_device_bytes": (_I64, [_P]),
    "shampoo_check_finite": (C.c_int, [_P, C.POINTER(_P), _I32, _P]),
    "shampoo_check_finite_deferred": (C.c_int, [_P, C.POINTER(_P), _I32, C.c_int64, C.POINTER(_I32), _P]),
    "shampoo_check_finite_resolve": (C.c_int, [_P, C.POINTER(_I32)]),
    "shampoo_gemm_timing": (C.c_int, [_I32, C.POINTER(_D), C.POINTER(_D), _PI64]),
    "shampoo_allgather": (C.c_int, [_P, _P, _P]),
    "shampoo_stats_update": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), _I32, _I64, _P]),
    "shampoo_root_inverse": (C.c_int, [_P, _I64, _PI32, _P]),
    "shampoo_pack_gradients": (C.c_int, [_P, C.POINTER(_P), _I32, _P, _P]),
    "shampoo_reduced_nonfinite": (C.c_int, [_P, _P, _P, _P]),
    "shampoo_stats_update_reduced": (C.c_int, [_P, _P, _D, C.POINTER(_P), _I32, _I64, _P]),
    "shampoo_precondition_graft": (C.c_int, [_P, C.POINTER(_P), _I32, _I64, _P]),
    "shampoo_apply": (C.c_int, [_P, C.POINTER(_P), _I32, _D, _P]),
    "shampoo_gather_buffer": (_P, [_P, _PI64, _PI32]),
    "shampoo_guard_stats_get": (C.c_int, [_P, C.POINTER(GuardStatsC)]),
    "shampoo_guard_stats_set": (C.c_int, [_P, C.POINTER(GuardStatsC)]),
    "shampoo_launch_count": (_I64, []),
    "shampoo_tc_counter": (C.c_int, [_I32, C.POINTER(C.c_double)]),
    "shampoo_timing_enable": (C.c_int, [_P, _I32]),
    "shampoo_timing_get": (C.c_int, [_P, C.POINTER(C.c_double), _PI64]),
    "shampoo_work": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "shampoo_work_tc": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]),
    "shampoo_state_view": (_P, [_P, _I32, C.c_char_p, _I32, _PI64, _PI32]),
    "shampoo_state_scalars_get": (C.c_int, [_P, _I32, _PI64, _PI64, _PI32]),
    "shampoo_state_scalars_set": (C.c_int, [_P, _I32, _I64, _I64, _I32]),
    "shampoo_graft_step_get": (C.c_int, [_P, _PI64]),
    "shampoo_graft_step_set": (C.c_int, [_P, _I64]),
    "shampoo_batched_root_inverse": (C.c_int, [C.POINTER(_P), C.POINTER(_P), _PI32, _I32, _I32, _D, _D,
                                               _I32, _D, _PI32, _PI32, _P]),
    "shampoo_tc_gemm": (C.c_int, [_P, _P, _P, _I32, _I32, _I32, _I32, _D, _D, _I32, _P]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libshampoo_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} not found: build it with `python -m paper_2309_06497_b200.build_native` "
                "(there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def last_error() -> str:
    return lib().shampoo_last_error().decode()


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = last_error()
    from .config import InvalidGroupSizeError, NonFiniteGradientError
    if rc == ERR_INVALID_GROUP:
        raise InvalidGroupSizeError(msg)
    if rc == ERR_NONFINITE_GRAD:
        raise NonFiniteGradientError(msg)
    if rc in (ERR_INVALID_ARGUMENT, ERR_SHAPE):
        raise ValueError(msg)
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise NativeError(f"{what}: {msg} (code {rc})")


def ptr_array(ptrs) -> "C.Array":
    arr = (C.c_void_p * max(len(ptrs), 1))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


class DeviceView:
    """Zero-copy torch view of library-owned device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, numel: int, f32: bool, owner=None):
        self.__cuda_array_interface__ = {
            "shape": (int(numel),),
            "typestr": "<f4" if f32 else "<f8",
            "data": (int(ptr), False),
            "version": 3,
            "strides": None,
        }
        self._owner = owner
