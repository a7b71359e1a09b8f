"""ctypes binding of libicv.so (C ABI declared in include/icv.h).

This is the Python side of the drop-in boundary: the public functions in
``indirect.py`` / ``gemm.py`` validate arguments exactly as the reference does
and then call these entry points with raw device pointers.  There is no CPU
fallback — if the library is missing or cannot be loaded every compute call
raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading

import torch

from .errors import InvalidGeometryError, NativeLibraryError, StaleBufferError, UnsupportedError  # noqa: F401

LIB_PATH = os.environ.get("ICV_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libicv.so")

ICV_OK, ICV_ERR_ARG, ICV_ERR_GEOMETRY, ICV_ERR_STALE, ICV_ERR_UNSUPPORTED, ICV_ERR_CUDA = 0, -1, -2, -3, -4, -5
ICV_F32, ICV_BF16, ICV_U8, ICV_I32, ICV_I64 = 0, 1, 2, 3, 4
ICV_IB_PER_IMAGE = 0x100
ICV_IB_CANONICAL = 0x200   # buffer is exactly icv_ib_build's output (row-sliding kernels may use it)
ICV_ZERO_ROW_ZEROS = 0x400  # bound zero row is all zero bytes (window kernels may zero-fill padding)
ICV_ZERO_ROW_ZP = 0x800     # uint8: every zero-row byte is the input zero point (zero fill + per-tap correction)
ICV_PREFER_GATHER = 0x1000  # run the IB-gather kernels (no window / row-sliding / dense-A specialisation)

TORCH_TO_ICV = {torch.float32: ICV_F32, torch.bfloat16: ICV_BF16, torch.uint8: ICV_U8,
                torch.int32: ICV_I32, torch.int64: ICV_I64}


class Desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "kernel_h", "kernel_w", "stride_h", "stride_w", "dilation_h", "dilation_w",
        "pad_top", "pad_left", "pad_bottom", "pad_right", "in_channels", "out_channels")]


class Shape(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("h", ctypes.c_int64), ("w", ctypes.c_int64), ("c", ctypes.c_int64)]


class Quant(ctypes.Structure):
    _fields_ = [("input_zero_point", ctypes.c_int32), ("input_scale", ctypes.c_float),
                ("kernel_zero_point", ctypes.c_int32), ("kernel_scale", ctypes.c_float),
                ("output_zero_point", ctypes.c_int32), ("output_scale", ctypes.c_float),
                ("output_min", ctypes.c_int32), ("output_max", ctypes.c_int32)]


# name -> (restype, argtypes); the full exported surface of include/icv.h
_P = ctypes.c_void_p
_I32, _I64, _F32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float
SIGNATURES = {
    "icv_abi_version": (_I32, []),
    "icv_last_error": (ctypes.c_char_p, []),
    "icv_device_info": (ctypes.c_int, [_I32, ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "icv_out_shape": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.POINTER(Shape), ctypes.POINTER(Shape)]),
    "icv_ib_entries": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.POINTER(Shape), _I64, _I32,
                                      ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "icv_ib_build": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.POINTER(Shape), _I64, _I32, _I64, _I32, _P, _P]),
    "icv_ib_check": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.POINTER(Shape), _I64, _I32, _I32, _P, _P, _P]),
    "icv_packed_filter_bytes": (ctypes.c_int, [ctypes.POINTER(Desc), _I32, ctypes.POINTER(_I64)]),
    "icv_pack_filter": (ctypes.c_int, [ctypes.POINTER(Desc), _I32, _I32, _P, _P, ctypes.POINTER(Quant), _P, _P]),
    "icv_requant_params": (ctypes.c_int, [_F32, _F32, _F32, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "icv_conv": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.POINTER(Shape), _I64, _I32, _P, _P, _P, _I32, _I32,
                                _P, ctypes.POINTER(Quant), _P, _P]),
    "icv_conv_kernel_name": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.POINTER(Shape), _I32, _I32,
                                            ctypes.POINTER(ctypes.c_char_p)]),
    "icv_set_tuning": (ctypes.c_int, [ctypes.c_char_p, _I32]),
    "icv_direct_conv": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.POINTER(Shape), _I64, _I32, _P, _I32, _P, _P,
                                        _P, _P]),
    "icv_nccl_version": (ctypes.c_int, [ctypes.POINTER(_I32)]),
    "icv_nccl_unique_id": (ctypes.c_int, [_P]),
    "icv_nccl_init_rank": (ctypes.c_int, [ctypes.POINTER(_P), _I32, _P, _I32]),
    "icv_nccl_init_all": (ctypes.c_int, [ctypes.POINTER(_P), _I32, ctypes.POINTER(_I32)]),
    "icv_nccl_comm_size": (ctypes.c_int, [_P, ctypes.POINTER(_I32)]),
    "icv_nccl_broadcast": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _P]),
    "icv_nccl_destroy": (ctypes.c_int, [_P]),
    "icv_get_tuning": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_I32)]),
    "icv_launch_count": (_I64, []),
    "icv_maxpool2d": (ctypes.c_int, [ctypes.POINTER(Shape), _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _P, _P]),
    "icv_im2col": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.POINTER(Shape), _I64, _I32, _P, _P, _P, _P]),
}

_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load libicv.so once; raise NativeLibraryError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryError(
                    f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            try:
                handle = ctypes.CDLL(LIB_PATH)
            except OSError as exc:  # pragma: no cover - depends on the box
                raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().icv_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str) -> None:
    """Map an icv_status to the reference's exception types."""
    if status == ICV_OK:
        return
    msg = f"{what}: {last_error()}"
    if status == ICV_ERR_GEOMETRY:
        raise InvalidGeometryError(msg)
    if status == ICV_ERR_ARG:
        raise ValueError(msg)
    if status == ICV_ERR_STALE:
        raise StaleBufferError(msg)
    if status == ICV_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise NativeLibraryError(msg)


def desc_of(params) -> Desc:
    return Desc(*(int(getattr(params, f)) for f, _ in Desc._fields_))


def shape_of(shape) -> Shape:
    return Shape(int(shape.n), int(shape.h), int(shape.w), int(shape.c))


def quant_of(q) -> Quant | None:
    if q is None:
        return None
    return Quant(int(q.input_zero_point), float(q.input_scale), int(q.kernel_zero_point), float(q.kernel_scale),
                 int(q.output_zero_point), float(q.output_scale), int(q.output_min), int(q.output_max))


def ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def stream_of(device: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def require_cuda(t: torch.Tensor, what: str) -> None:
    if t.device.type != "cuda":
        raise NativeLibraryError(
            f"{what} must live in CUDA device memory (got {t.device}); the B200 path has no CPU fallback")


def launch_count() -> int:
    return int(lib().icv_launch_count())


DEFAULT_FLAGS = ICV_IB_CANONICAL | ICV_ZERO_ROW_ZEROS | ICV_IB_PER_IMAGE


def kernel_name(params, in_shape, dtype: torch.dtype, flags: int | None = None) -> str:
    """Kernel icv_conv launches for this problem; ``flags`` are the layout
    flags of its ``ib_dtype`` argument (default: a canonical per-image buffer
    with a zero zero row, as init_indirection_buffer / make_zero_row build;
    uint8 adds ICV_ZERO_ROW_ZP when the zero row holds the zero point)."""
    out = ctypes.c_char_p()
    d, s = desc_of(params), shape_of(in_shape)
    if flags is None:
        flags = DEFAULT_FLAGS if dtype != torch.uint8 else (ICV_IB_CANONICAL | ICV_IB_PER_IMAGE | ICV_ZERO_ROW_ZP)
    f = int(flags)
    check(lib().icv_conv_kernel_name(ctypes.byref(d), ctypes.byref(s), TORCH_TO_ICV[dtype], f, ctypes.byref(out)),
          "icv_conv_kernel_name")
    return out.value.decode()


def set_tuning(key: str, value: int) -> None:
    """Set a plan knob of the native library (include/icv.h icv_set_tuning)."""
    check(lib().icv_set_tuning(key.encode(), int(value)), "icv_set_tuning")


def get_tuning(key: str) -> int:
    v = _I32()
    check(lib().icv_get_tuning(key.encode(), ctypes.byref(v)), "icv_get_tuning")
    return int(v.value)


@contextlib.contextmanager
def tuning(**knobs):
    """Temporarily set plan knobs (A/B measurement, tests); restored on exit."""
    saved = {k: get_tuning(k) for k in knobs}
    try:
        for k, v in knobs.items():
            set_tuning(k, v)
        yield
    finally:
        for k, v in saved.items():
            set_tuning(k, v)
