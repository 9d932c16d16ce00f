"""ctypes binding of libmoqe_gpu.so — the C-ABI declared in include/moqe_gpu.h.

The library is built in-tree (paper_2310_02410_b200/lib/libmoqe_gpu.so) by
``build.build()``. Loading fails loudly if it is missing: there is no CPU or
eager fallback for any operation of this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MOQE_GPU_LIB: an alternate build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("MOQE_GPU_LIB") or os.path.join(HERE, "lib", "libmoqe_gpu.so")

# status codes (moqe_status)
OK, INVALID_ARGUMENT, OUT_OF_RANGE, RANGE_ERROR, CUDA_ERROR, NCCL_ERROR, NOT_SUPPORTED, CHECKPOINT_ERROR = range(8)
PER_CHANNEL, PER_TENSOR = 0, 1
SCHEME_LINEAR, SCHEME_LOG = 0, 1
F32, F16 = 0, 1
PATH_AUTO, PATH_GEMV, PATH_GEMM = 0, 1, 2

# Every symbol include/moqe_gpu.h declares: (restype, argtypes)
_vp, _i64, _i32, _sz = C.c_void_p, C.c_int64, C.c_int, C.c_size_t
SIGNATURES = {
    "moqe_gpu_abi_version": (_i32, []),
    "moqe_gpu_last_error": (C.c_char_p, []),
    "moqe_gpu_status_string": (C.c_char_p, [_i32]),
    "moqe_gpu_packed_size": (_sz, [_i32, _sz]),
    "moqe_gpu_pack": (_i32, [_vp, _i64, _i32, _vp, _vp]),
    "moqe_gpu_unpack": (_i32, [_vp, _i64, _i32, _i64, _vp, _vp]),
    "moqe_gpu_linear_scales": (_i32, [_vp, _i64, _i64, _i64, _i32, _i32, _vp, _vp]),
    "moqe_gpu_quantize_linear": (_i32, [_vp, _i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp]),
    "moqe_gpu_quantize_pack": (_i32, [_vp, _i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp]),
    "moqe_gpu_route": (_i32, [_vp, _i32, _i64, _i64, _vp, _i32, _i32, _vp, _vp, _vp]),
    "moqe_gpu_bank_create": (_i32, [_i32, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32,
                                    C.POINTER(_vp)]),
    "moqe_gpu_bank_create_g": (_i32, [_i32, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32,
                                      C.POINTER(_vp)]),
    "moqe_gpu_bank_create_ex": (_i32, [_i32, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32,
                                       C.POINTER(_vp)]),
    "moqe_gpu_bank_destroy": (_i32, [_vp]),
    "moqe_gpu_bank_set_router": (_i32, [_vp, _vp, _i32]),
    "moqe_gpu_bank_weight_bytes": (_i64, [_vp]),
    "moqe_gpu_moe_forward": (_i32, [_vp, _vp, _i32, _i64, _vp, _i32, _vp, _i32, _vp, _vp, _i32,
                                    _vp]),
    "moqe_gpu_expert_ffn": (_i32, [_vp, _vp, _i32, _i64, _vp, _vp, _vp, _i32, _i32, _vp]),
    "moqe_gpu_bank_profile": (_i32, [_vp, _i32]),
    "moqe_gpu_bank_profile_read": (_i32, [_vp, _vp, _vp, _i32]),
    "moqe_gpu_mqe1_open": (_i32, [C.c_char_p, C.POINTER(_vp)]),
    "moqe_gpu_mqe1_close": (_i32, [_vp]),
    "moqe_gpu_mqe1_count": (_i64, [_vp]),
    "moqe_gpu_mqe1_entry": (_i32, [_vp, _i64, _vp]),
    "moqe_gpu_mqe1_bank_create": (_i32, [_vp, C.c_char_p, _i32, C.POINTER(_vp)]),
    "moqe_gpu_add_layer_norm": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _i32, _vp]),
    "moqe_gpu_bank_span": (_i32, [_vp, _i32]),
    "moqe_gpu_bank_span_read": (_i32, [_vp, _vp, _vp]),
    "moqe_gpu_bank_trace": (_i32, [_vp, _i32]),
    "moqe_gpu_bank_trace_read": (_i64, [_vp, _vp, _i64]),
    "moqe_gpu_moe_forward_host": (_i32, [_vp, _vp, _i32, _i64, _i32, _vp, _i32, _vp]),
    "moqe_gpu_ep_dispatch": (_i32, [_vp, _i64, _i64, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "moqe_gpu_ep_combine": (_i32, [_vp, _i32, _vp, _i64, _i32, _i64, _vp, _vp]),
}


class MoqeError(RuntimeError):
    """Base class; subclasses mirror the reference's exception types."""


class InvalidArgument(MoqeError, ValueError):
    """std::invalid_argument in the reference."""


class OutOfRange(MoqeError, IndexError):
    """std::out_of_range in the reference (bitpack.cpp:27-29)."""


class RangeError(MoqeError, ArithmeticError):
    """std::range_error in the reference (tensor.cpp:101-104)."""


class CheckpointError(MoqeError, RuntimeError):
    """moqe::CheckpointError in the reference (checkpoint.hpp:14-30)."""


class CudaError(MoqeError):
    pass


class NotSupported(MoqeError):
    pass


_EXC = {INVALID_ARGUMENT: InvalidArgument, OUT_OF_RANGE: OutOfRange, RANGE_ERROR: RangeError,
        CUDA_ERROR: CudaError, NCCL_ERROR: MoqeError, NOT_SUPPORTED: NotSupported,
        CHECKPOINT_ERROR: CheckpointError}

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the C-ABI library (no GPU needed to load it)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} is not built; run paper_2310_02410_b200.build.build() "
                              "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status != OK:
        lib = load()
        msg = lib.moqe_gpu_last_error().decode(errors="replace")
        raise _EXC.get(status, MoqeError)(msg)
