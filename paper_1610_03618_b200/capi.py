"""ctypes binding of the C ABI declared in include/lcnn_cuda.h.

This is the reference-side binding a Python maintainer would add (see
INTEGRATION.md).  It loads the in-tree sm_100a library
``paper_1610_03618_b200/lib/liblcnn_cuda.so`` and fails loudly if it is
missing: there is no CPU or eager-PyTorch fallback anywhere in the product
path.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_size_t, c_uint32, c_uint64, c_void_p

from .errors import raise_for_status

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "lib", "liblcnn_cuda.so")
HEADER_PATH = os.path.join(os.path.dirname(PKG_DIR), "include", "lcnn_cuda.h")

# lcnn_layout / lcnn_pool_mode codes (tensor.hpp:16, pool.hpp:11)
NCHW, CHWN, NHWC, HWCN = 0, 1, 2, 3
LAYOUT_NAMES = {NCHW: "nchw", CHWN: "chwn", NHWC: "nhwc", HWCN: "hwcn"}
POOL_MAX, POOL_AVG = 0, 1
PREC_TF32, PREC_3XTF32, PREC_FP32 = 0, 1, 2


class AccessReport(ctypes.Structure):
    """== lcnn::AccessReport (pool.hpp:30-34)."""

    _fields_ = [("input_loads", c_uint64), ("output_stores", c_uint64),
                ("distinct_inputs", c_uint64)]

    def as_tuple(self):
        return (self.input_loads, self.output_stores, self.distinct_inputs)


class PoolPlan(ctypes.Structure):
    """== lcnn_pool_plan (include/lcnn_cuda.h): a pooling kernel plan."""

    _fields_ = [("fh", c_uint32), ("fw", c_uint32), ("ring_kb", c_uint32),
                ("ring_slots", c_uint32), ("ring_ctas", c_uint32), ("tuned", c_int),
                ("us", ctypes.c_float)]

    def as_tuple(self):
        return (self.fh, self.fw, self.ring_kb, self.ring_slots, self.ring_ctas)

    def __repr__(self):
        ring = f" ring={self.ring_kb}KBx{self.ring_slots}x{self.ring_ctas}" if self.ring_kb else ""
        return f"PoolPlan({self.fh}x{self.fw}{ring}{' tuned' if self.tuned else ''})"


class PassReport(ctypes.Structure):
    """== lcnn::PassReport (softmax.hpp:21-24)."""

    _fields_ = [("materializations", c_uint32), ("full_matrix_sweeps", c_uint32)]


_U32 = c_uint32
_P = c_void_p
_SIGNATURES = {
    "lcnn_abi_version": (c_int, []),
    "lcnn_last_error": (c_char_p, []),
    "lcnn_status_name": (c_char_p, [c_int]),
    "lcnn_device_ok": (c_int, []),
    "lcnn_flattenable_pair": (c_int, [c_int, c_int]),
    "lcnn_transform": (c_int, [_P, _P, _U32, _U32, _U32, _U32, c_int, c_int, _P]),
    "lcnn_transform_tiled": (c_int, [_P, _P, _U32, _U32, _U32, _U32, c_int, c_int, _U32, c_int, _P]),
    "lcnn_transform_naive": (c_int, [_P, _P, _U32, _U32, _U32, _U32, c_int, c_int, _P]),
    "lcnn_pool_output_extents": (c_int, [_U32, _U32, _U32, _U32, _U32, POINTER(_U32), POINTER(_U32)]),
    "lcnn_pool_layout": (c_int, [_P, _P, _U32, _U32, _U32, _U32, c_int, _U32, _U32, _U32, c_int,
                                 POINTER(AccessReport), _P]),
    "lcnn_pool_coarsened": (c_int, [_P, _P, _U32, _U32, _U32, _U32, c_int, _U32, _U32, _U32, c_int,
                                    _U32, _U32, POINTER(AccessReport), _P]),
    "lcnn_pool_coarsened_nchw": (c_int, [_P, _P, _U32, _U32, _U32, _U32, _U32, _U32, _U32, c_int,
                                         _U32, _U32, POINTER(AccessReport), _P]),
    "lcnn_pool_tune": (c_int, [_U32] * 4 + [c_int] + [_U32] * 3 + [c_int, POINTER(PoolPlan), _P]),
    "lcnn_pool_plan_lookup": (c_int, [_U32] * 4 + [c_int] + [_U32] * 3 + [c_int,
                                                                      POINTER(PoolPlan)]),
    "lcnn_pool_run_plan": (c_int, [_P, _P] + [_U32] * 4 + [c_int] + [_U32] * 3 +
                           [c_int, POINTER(PoolPlan), POINTER(AccessReport), _P]),
    "lcnn_pool_oracle": (c_int, [_P, _P, _U32, _U32, _U32, _U32, c_int, _U32, _U32, _U32, c_int, _P]),
    "lcnn_softmax_fused": (c_int, [_P, _P, _U32, _U32, _U32, _P, POINTER(PassReport), _P]),
    "lcnn_softmax_fused_sticky": (c_int, [_P, _P, _U32, _U32, _P, _P]),
    "lcnn_softmax_reference_scratch_bytes": (c_size_t, [_U32, _U32]),
    "lcnn_softmax_reference": (c_int, [_P, _P, _U32, _U32, _P, c_size_t, _P, POINTER(PassReport), _P]),
    "lcnn_conv_output_extents": (c_int, [_U32, _U32, _U32, _U32, _U32, _U32, POINTER(_U32),
                                         POINTER(_U32)]),
    "lcnn_conv_workspace_bytes": (c_size_t, [_U32] * 7 + [c_int]),
    "lcnn_conv_workspace_bytes_ex": (c_size_t, [_U32] * 4 + [c_int] + [_U32] * 5 + [c_int]),
    "lcnn_conv_forward": (c_int, [_P, _P, _P, _U32, _U32, _U32, _U32, c_int, _U32, _U32, _U32, _U32,
                                  _U32, c_int, _P, c_size_t, _P]),
    "lcnn_conv_packed_bytes": (c_size_t, [_U32] * 4 + [c_int] + [_U32] * 5 + [c_int]),
    "lcnn_conv_packed_workspace_bytes": (c_size_t, [_U32] * 4 + [c_int] + [_U32] * 5 + [c_int]),
    "lcnn_conv_pack_filters": (c_int, [_P, _P, c_size_t] + [_U32] * 4 + [c_int] + [_U32] * 5 +
                               [c_int, _P]),
    "lcnn_conv_forward_packed": (c_int, [_P, _P, _P] + [_U32] * 4 + [c_int] + [_U32] * 5 +
                                 [c_int, _P, c_size_t, _P]),
    "lcnn_conv_forward_packed_ex": (c_int, [_P, _P, _P] + [_U32] * 4 + [c_int] + [_U32] * 5 +
                                    [c_int, _P, c_size_t, _P, _P]),
    "lcnn_conv_maxpool_supported": (c_int, [_U32] * 4 + [c_int] + [_U32] * 5 + [c_int] +
                                    [_U32] * 2),
    "lcnn_conv_maxpool_packed": (c_int, [_P, _P, _P] + [_U32] * 4 + [c_int] + [_U32] * 5 +
                                 [c_int] + [_U32] * 2 + [_P]),
    "lcnn_conv_hwcn32_supported": (c_int, [_U32] * 4 + [_U32] * 5 + [c_int] + [_U32] * 3),
    "lcnn_conv_forward_packed_blk": (c_int, [_P, _P, _P] + [_U32] * 4 + [c_int] + [_U32] * 5 +
                                     [c_int, _P, c_size_t, _P, _U32, _P]),
    "lcnn_conv_maxpool_packed_blk": (c_int, [_P, _P, _P] + [_U32] * 4 + [c_int] + [_U32] * 5 +
                                     [c_int] + [_U32] * 3 + [_P]),
    "lcnn_conv_oracle": (c_int, [_P, _P, _P, _U32, _U32, _U32, _U32, c_int, _U32, _U32, _U32, _U32,
                                 _U32, _P]),
    "lcnn_im2col": (c_int, [_P, _P, _U32, _U32, _U32, _U32, c_int, _U32, _U32, _U32, _U32, _P]),
    "lcnn_gemm_workspace_bytes": (c_size_t, [c_uint64, c_uint64, c_uint64, c_int]),
    "lcnn_gemm": (c_int, [_P, _P, _P, c_uint64, c_uint64, c_uint64, c_int, _P, c_size_t, _P]),
    "lcnn_fc_packed_bytes": (c_size_t, [c_uint64, c_uint64, c_int]),
    "lcnn_fc_workspace_bytes": (c_size_t, [c_uint64, c_uint64, c_int]),
    "lcnn_fc_pack_weights": (c_int, [_P, _P, c_size_t, c_uint64, c_uint64, c_int, _P]),
    "lcnn_fc_forward_packed": (c_int, [_P, c_int, _P, _P, c_uint64, c_uint64, c_uint64, c_int, _P,
                                       c_size_t, _P]),
    "lcnn_fc_forward_packed_ex": (c_int, [_P, c_int, _P, _P, c_uint64, c_uint64, c_uint64, c_int,
                                          _P, c_size_t, _P, _P, c_size_t, _P]),
}
SYNC_BYTES = 16  # LCNN_SYNC_BYTES

_lib = None


def lib() -> ctypes.CDLL:
    """Load the CUDA library once; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"lcnn CUDA library missing at {LIB_PATH}: run `python -c 'import "
                "__graft_entry__ as g; g.build()'` (or `make`) first -- there is no "
                "CPU fallback")
        dll = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(dll, name)
            fn.restype = res
            fn.argtypes = args
        _lib = dll
    return _lib


def declared_symbols(header: str = HEADER_PATH) -> list[str]:
    """Every function name declared in include/lcnn_cuda.h."""
    import re

    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lcnn_[a-z0-9_]+)\s*\(", text)))


def check(status: int, where: str = "") -> None:
    """Raise the lcnn exception matching a non-zero status."""
    if status:
        msg = lib().lcnn_last_error().decode()
        raise_for_status(status, msg or where)


def call(name: str, *args) -> int:
    st = getattr(lib(), name)(*args)
    check(st, name)
    return st


__all__ = [
    "AccessReport", "PassReport", "PoolPlan", "lib", "call", "check", "declared_symbols", "LIB_PATH",
    "NCHW", "CHWN", "NHWC", "HWCN", "POOL_MAX", "POOL_AVG", "PREC_TF32", "PREC_3XTF32",
    "LAYOUT_NAMES", "c_double", "PREC_FP32", "SYNC_BYTES",
]
