"""Device-resident mirror of the reference operator API over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/lcnn/{tensor,layout,pool,softmax,select}.hpp so
the parity tests read like the reference's own tests.  Tensors live in HBM
(PyTorch is used only to own device memory and streams); every op is one call
into liblcnn_cuda.so on the current CUDA stream.  Whole networks (parse,
annotate, device-resident forward, host-buffer forwards) are in
:mod:`paper_1610_03618_b200.netapi` over liblcnn.so (include/lcnn_net.h).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import CHWN, HWCN, NCHW, NHWC, POOL_AVG, POOL_MAX, AccessReport, PassReport
from .errors import DomainError, ShapeError

K_COARSENING_CAP = 64  # pool.hpp:28


def _torch():
    import torch

    return torch


def _stream(stream=None) -> int:
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    return _torch().cuda.current_stream().cuda_stream


def layout_strides(layout: int, n: int, c: int, h: int, w: int) -> tuple[int, int, int, int]:
    """== layout_strides (tensor.cpp:55-85): (sn, sc, sh, sw)."""
    if layout == NCHW:
        return (c * h * w, h * w, w, 1)
    if layout == CHWN:
        return (1, h * w * n, w * n, n)
    if layout == NHWC:
        return (h * w * c, 1, w * c, c)
    return (1, n, w * c * n, c * n)  # HWCN


def _check_volume(n, c, h, w, what="Tensor4D"):
    if min(n, c, h, w) < 1:
        raise ShapeError(f"{what}: all dims must be >= 1")
    if n * c * h * w > 0xFFFFFFFF:
        raise ShapeError(f"{what}: dim product overflows")


@dataclass
class DeviceTensor4D:
    """Dense fp32 4D tensor in HBM tagged with its layout (tensor.hpp:33-73)."""

    n: int
    c: int
    h: int
    w: int
    layout: int
    data: "object"  # torch.Tensor, 1-D float32 on a CUDA device

    @staticmethod
    def empty(n, c, h, w, layout, device="cuda"):
        _check_volume(n, c, h, w)
        t = _torch().empty(n * c * h * w, dtype=_torch().float32, device=device)
        return DeviceTensor4D(n, c, h, w, layout, t)

    @staticmethod
    def from_host(arr, n, c, h, w, layout, device="cuda"):
        _check_volume(n, c, h, w)
        a = np.ascontiguousarray(arr, dtype=np.float32).reshape(-1)
        if a.size != n * c * h * w:
            raise ShapeError("Tensor4D: data length does not match dims")
        return DeviceTensor4D(n, c, h, w, layout, _torch().from_numpy(a).to(device))

    def to_host(self) -> np.ndarray:
        return self.data.detach().cpu().numpy()

    @property
    def size(self) -> int:
        return self.n * self.c * self.h * self.w

    def strides(self):
        return layout_strides(self.layout, self.n, self.c, self.h, self.w)

    def ptr(self) -> int:
        return self.data.data_ptr()

    def with_layout_tag(self, layout):
        """Same buffer under a different tag (tensor.hpp:70)."""
        return DeviceTensor4D(self.n, self.c, self.h, self.w, layout, self.data)

    def same_dims(self, o) -> bool:
        return (self.n, self.c, self.h, self.w) == (o.n, o.c, o.h, o.w)


@dataclass
class DeviceMatrix:
    """Row-major fp32 matrix in HBM (tensor.hpp:106-121)."""

    rows: int
    cols: int
    data: "object"

    @staticmethod
    def empty(rows, cols, device="cuda"):
        return DeviceMatrix(rows, cols, _torch().empty(rows * cols, dtype=_torch().float32, device=device))

    @staticmethod
    def from_host(arr, rows, cols, device="cuda"):
        a = np.ascontiguousarray(arr, dtype=np.float32).reshape(-1)
        if a.size != rows * cols:
            raise ShapeError("Matrix: data length does not match dims")
        return DeviceMatrix(rows, cols, _torch().from_numpy(a).to(device))

    def to_host(self) -> np.ndarray:
        return self.data.detach().cpu().numpy()

    def ptr(self) -> int:
        return self.data.data_ptr()


# ---------------------------------------------------------------- layout --
TILED_2D, NAIVE_PERMUTE = 0, 1


@dataclass
class TransformPlan:
    """== TransformPlan (layout.hpp:16-22)."""

    src: int = NCHW
    dst: int = NCHW
    tile: int = 32
    wide_copy: bool = False
    kind: int = TILED_2D


def flattenable_pair(src: int, dst: int) -> bool:
    return bool(capi.lib().lcnn_flattenable_pair(src, dst))


def make_plan(src, dst, n, c, h, w) -> TransformPlan:
    """== make_plan (layout.cpp:122-136)."""
    if flattenable_pair(src, dst):
        return TransformPlan(src, dst, 32, n >= 64, TILED_2D)
    return TransformPlan(src, dst, 32, False, NAIVE_PERMUTE)


def _out4(t: DeviceTensor4D, layout, out):
    if out is None:
        return DeviceTensor4D(t.n, t.c, t.h, t.w, layout,
                              _torch().empty(t.size, dtype=_torch().float32, device=t.data.device))
    if not out.same_dims(t) or out.size != t.size:
        raise ShapeError("transform: output dims do not match")
    out.layout = layout
    return out


def transform_naive(t: DeviceTensor4D, dst: int, out=None, stream=None) -> DeviceTensor4D:
    o = _out4(t, dst, out)
    capi.call("lcnn_transform_naive", t.ptr(), o.ptr(), t.n, t.c, t.h, t.w, t.layout, dst,
              _stream(stream))
    return o


def transform_tiled(t: DeviceTensor4D, dst: int, plan: TransformPlan, out=None,
                    stream=None) -> DeviceTensor4D:
    from .errors import PlanError

    if plan.dst != dst:
        raise PlanError("transform_tiled: plan destination layout does not match")
    if plan.src != t.layout:
        raise PlanError("transform_tiled: plan source layout does not match tensor")
    o = _out4(t, dst, out)
    capi.call("lcnn_transform_tiled", t.ptr(), o.ptr(), t.n, t.c, t.h, t.w, t.layout, dst,
              plan.tile, int(plan.wide_copy), _stream(stream))
    return o


def transform(t: DeviceTensor4D, dst: int, out=None, stream=None) -> DeviceTensor4D:
    """== transform (layout.cpp:138-144)."""
    o = _out4(t, dst, out)
    capi.call("lcnn_transform", t.ptr(), o.ptr(), t.n, t.c, t.h, t.w, t.layout, dst,
              _stream(stream))
    return o


# ------------------------------------------------------------------ pool --
MAX, AVERAGE = POOL_MAX, POOL_AVG


@dataclass
class PoolParams:
    """== PoolParams (pool.hpp:13-18)."""

    win_h: int = 2
    win_w: int = 2
    stride: int = 2
    mode: int = MAX


@dataclass
class CoarseningPlan:
    fh: int = 1
    fw: int = 1


def pool_output_extents(h, w, p: PoolParams):
    ho, wo = ctypes.c_uint32(), ctypes.c_uint32()
    capi.call("lcnn_pool_output_extents", h, w, p.win_h, p.win_w, p.stride,
              ctypes.byref(ho), ctypes.byref(wo))
    return ho.value, wo.value


def _pool_out(t, p, layout, out):
    if p.win_h < 1 or p.win_w < 1 or p.stride < 1 or p.win_h > t.h or p.win_w > t.w:
        # let the library produce the reference's exact error
        ho = wo = 1
    else:
        ho, wo = (t.h - p.win_h) // p.stride + 1, (t.w - p.win_w) // p.stride + 1
    if out is None:
        out = DeviceTensor4D(t.n, t.c, ho, wo, layout,
                             _torch().empty(t.n * t.c * ho * wo, dtype=_torch().float32,
                                            device=t.data.device))
    return out


def pool_layout(t: DeviceTensor4D, p: PoolParams, out=None, stream=None):
    """== pool_layout (pool.cpp:172-176) -> (output, AccessReport)."""
    o = _pool_out(t, p, t.layout, out)
    rep = AccessReport()
    capi.call("lcnn_pool_layout", t.ptr(), o.ptr(), t.n, t.c, t.h, t.w, t.layout, p.win_h,
              p.win_w, p.stride, p.mode, ctypes.byref(rep), _stream(stream))
    return o, rep


def pool_coarsened(t: DeviceTensor4D, p: PoolParams, plan: CoarseningPlan, out=None,
                   stream=None):
    """== pool_coarsened (pool.cpp:178-270) -> (output, AccessReport)."""
    o = _pool_out(t, p, CHWN, out)
    rep = AccessReport()
    capi.call("lcnn_pool_coarsened", t.ptr(), o.ptr(), t.n, t.c, t.h, t.w, t.layout, p.win_h,
              p.win_w, p.stride, p.mode, plan.fh, plan.fw, ctypes.byref(rep), _stream(stream))
    return o, rep


def pool_coarsened_nchw(t: DeviceTensor4D, p: PoolParams, plan: CoarseningPlan, out=None,
                        stream=None):
    """GPU extension: register-coarsened NCHW kernel (see lcnn_cuda.h)."""
    o = _pool_out(t, p, NCHW, out)
    rep = AccessReport()
    capi.call("lcnn_pool_coarsened_nchw", t.ptr(), o.ptr(), t.n, t.c, t.h, t.w, p.win_h,
              p.win_w, p.stride, p.mode, plan.fh, plan.fw, ctypes.byref(rep), _stream(stream))
    return o, rep


def pool_tune(n, c, h, w, layout, p: PoolParams, stream=None) -> "capi.PoolPlan":
    """GPU autotuner (lcnn_pool_tune): measure the layout's kernel plans for
    this shape, cache and return the fastest.  Afterwards pool_layout on the
    shape runs the tuned plan."""
    plan = capi.PoolPlan()
    capi.call("lcnn_pool_tune", n, c, h, w, layout, p.win_h, p.win_w, p.stride, p.mode,
              ctypes.byref(plan), _stream(stream))
    return plan


def pool_plan_lookup(n, c, h, w, layout, p: PoolParams) -> "capi.PoolPlan":
    plan = capi.PoolPlan()
    capi.call("lcnn_pool_plan_lookup", n, c, h, w, layout, p.win_h, p.win_w, p.stride, p.mode,
              ctypes.byref(plan))
    return plan


def pool_run_plan(t: DeviceTensor4D, p: PoolParams, plan, out=None, stream=None):
    """Pool with an explicit kernel plan (either layout) -> (output, AccessReport)."""
    o = _pool_out(t, p, t.layout, out)
    rep = AccessReport()
    capi.call("lcnn_pool_run_plan", t.ptr(), o.ptr(), t.n, t.c, t.h, t.w, t.layout, p.win_h,
              p.win_w, p.stride, p.mode, ctypes.byref(plan), ctypes.byref(rep), _stream(stream))
    return o, rep


def pool_oracle(t: DeviceTensor4D, p: PoolParams, out=None, stream=None):
    """== pool_oracle (pool.cpp:49-84): fp64, NCHW out."""
    o = _pool_out(t, p, NCHW, out)
    capi.call("lcnn_pool_oracle", t.ptr(), o.ptr(), t.n, t.c, t.h, t.w, t.layout, p.win_h,
              p.win_w, p.stride, p.mode, _stream(stream))
    return o


# --------------------------------------------------------------- softmax --
_flags: dict = {}


def _flag(device):
    key = str(device)
    if key not in _flags:
        _flags[key] = _torch().zeros(1, dtype=_torch().int32, device=device)
    return _flags[key]


def softmax_fused(m: DeviceMatrix, local_buffer_limit: int = 16384, out=None, check=True,
                  stream=None):
    """== softmax_fused (softmax.cpp:100-180) -> (output, PassReport).

    With check=True the non-finite flag is read back (one 4-byte D2H, which
    synchronises the stream) and DomainError raised as softmax.cpp:15-19 does.
    """
    if m.rows < 1 or m.cols < 1:
        raise ShapeError("softmax: empty matrix")
    o = out if out is not None else DeviceMatrix.empty(m.rows, m.cols, m.data.device)
    rep = PassReport()
    flag = _flag(m.data.device) if check else None
    capi.call("lcnn_softmax_fused", m.ptr(), o.ptr(), m.rows, m.cols, local_buffer_limit,
              flag.data_ptr() if flag is not None else None, ctypes.byref(rep), _stream(stream))
    if flag is not None and int(flag.item()):
        raise DomainError("softmax: non-finite input")
    return o, rep


def softmax_reference(m: DeviceMatrix, out=None, scratch=None, check=True, stream=None):
    """== softmax_reference (softmax.cpp:36-98): the five-kernel path."""
    if m.rows < 1 or m.cols < 1:
        raise ShapeError("softmax: empty matrix")
    o = out if out is not None else DeviceMatrix.empty(m.rows, m.cols, m.data.device)
    nbytes = capi.lib().lcnn_softmax_reference_scratch_bytes(m.rows, m.cols)
    if scratch is None:
        scratch = _torch().empty(nbytes // 4, dtype=_torch().float32, device=m.data.device)
    rep = PassReport()
    flag = _flag(m.data.device) if check else None
    capi.call("lcnn_softmax_reference", m.ptr(), o.ptr(), m.rows, m.cols, scratch.data_ptr(),
              scratch.numel() * 4, flag.data_ptr() if flag is not None else None,
              ctypes.byref(rep), _stream(stream))
    if flag is not None and int(flag.item()):
        raise DomainError("softmax: non-finite input")
    return o, rep


# ------------------------------------------------------- conv / gemm ------
TF32, X3TF32, FP32 = capi.PREC_TF32, capi.PREC_3XTF32, capi.PREC_FP32


def conv_output_extents(h, w, fh, fw, stride, pad):
    ho, wo = ctypes.c_uint32(), ctypes.c_uint32()
    capi.call("lcnn_conv_output_extents", h, w, fh, fw, stride, pad, ctypes.byref(ho),
              ctypes.byref(wo))
    return ho.value, wo.value


def conv_forward(x: DeviceTensor4D, filters, c_o, f_h, f_w, stride=1, pad=0, precision=FP32,
                 out=None, workspace=None, stream=None) -> DeviceTensor4D:
    """conv_direct (CHWN) / conv_gemm (NCHW) on the GPU; filters is a CUDA
    float32 tensor in (c_o, c_i, f_h, f_w) order (tensor.hpp:77-103)."""
    torch = _torch()
    ho, wo = conv_output_extents(x.h, x.w, f_h, f_w, stride, pad)
    if out is None:
        out = DeviceTensor4D(x.n, c_o, ho, wo, x.layout,
                             torch.empty(x.n * c_o * ho * wo, dtype=torch.float32,
                                         device=x.data.device))
    nbytes = capi.lib().lcnn_conv_workspace_bytes_ex(x.n, x.c, x.h, x.w, x.layout, c_o, f_h, f_w,
                                                     stride, pad, precision)
    if workspace is None or workspace.numel() * 4 < nbytes:
        workspace = torch.empty(max(1, (nbytes + 3) // 4), dtype=torch.float32,
                                device=x.data.device)
    capi.call("lcnn_conv_forward", x.ptr(), filters.data_ptr(), out.ptr(), x.n, x.c, x.h, x.w,
              x.layout, c_o, f_h, f_w, stride, pad, precision, workspace.data_ptr(),
              workspace.numel() * 4, _stream(stream))
    return out


def pack_conv_filters(x: DeviceTensor4D, filters, c_o, f_h, f_w, stride=1, pad=0,
                      precision=FP32, stream=None):
    """The filters packed into the operand image of the kernel x's geometry
    routes to (lcnn_conv_pack_filters) -> a CUDA uint8 tensor."""
    torch = _torch()
    geo = (x.n, x.c, x.h, x.w, x.layout, c_o, f_h, f_w, stride, pad, precision)
    nbytes = capi.lib().lcnn_conv_packed_bytes(*geo)
    if nbytes == 0:
        conv_output_extents(x.h, x.w, f_h, f_w, stride, pad)  # raises the geometry error
        raise ValueError("conv: no packed image for this geometry")
    packed = torch.empty(nbytes, dtype=torch.uint8, device=x.data.device)
    capi.call("lcnn_conv_pack_filters", filters.data_ptr(), packed.data_ptr(), nbytes, *geo,
              _stream(stream))
    return packed


def conv_forward_packed(x: DeviceTensor4D, packed, c_o, f_h, f_w, stride=1, pad=0,
                        precision=FP32, out=None, stream=None, sync=None,
                        blk=0) -> DeviceTensor4D:
    """conv_forward on filters made by pack_conv_filters for this geometry.
    sync: optional CUDA tensor of >= capi.SYNC_BYTES zeroed bytes owned by
    this call site (lcnn_conv_forward_packed_ex: in-kernel stream-K zeroing).
    blk = OUT_HWCN32: the output is written in the run_network-internal
    blocked [N/32][H][W][C][32] layout (lcnn_conv_forward_packed_blk)."""
    torch = _torch()
    ho, wo = conv_output_extents(x.h, x.w, f_h, f_w, stride, pad)
    if out is None:
        out = DeviceTensor4D(x.n, c_o, ho, wo, x.layout,
                             torch.empty(x.n * c_o * ho * wo, dtype=torch.float32,
                                         device=x.data.device))
    geo = (x.n, x.c, x.h, x.w, x.layout, c_o, f_h, f_w, stride, pad, precision)
    nbytes = capi.lib().lcnn_conv_packed_workspace_bytes(*geo)
    ws = torch.empty(max(1, (nbytes + 3) // 4), dtype=torch.float32, device=x.data.device)
    capi.call("lcnn_conv_forward_packed_blk", x.ptr(), packed.data_ptr(), out.ptr(), *geo,
              ws.data_ptr(), ws.numel() * 4, sync.data_ptr() if sync is not None else None,
              blk, _stream(stream))
    return out


IN_HWCN32, OUT_HWCN32 = 1, 2  # lcnn_cuda.h LCNN_CONV_IN_HWCN32 / LCNN_CONV_OUT_HWCN32


def conv_hwcn32_supported(x: DeviceTensor4D, c_o, f_h, f_w, stride, pad, precision, pool_win,
                          pool_stride, blk) -> bool:
    """lcnn_conv_hwcn32_supported: this CHWN layer's route reads (IN) or
    writes (OUT) the blocked layout."""
    return capi.lib().lcnn_conv_hwcn32_supported(
        x.n, x.c, x.h, x.w, c_o, f_h, f_w, stride, pad, precision, pool_win, pool_stride,
        blk) == 1


def conv_maxpool_supported(x: DeviceTensor4D, c_o, f_h, f_w, stride, pad, precision, pool_win,
                           pool_stride) -> bool:
    """lcnn_conv_maxpool_supported: the fused conv -> max-pool kernel covers
    this layer pair."""
    return capi.lib().lcnn_conv_maxpool_supported(
        x.n, x.c, x.h, x.w, x.layout, c_o, f_h, f_w, stride, pad, precision, pool_win,
        pool_stride) == 1


def conv_maxpool_packed(x: DeviceTensor4D, packed, c_o, f_h, f_w, stride, pad, precision,
                        pool_win, pool_stride, out=None, stream=None, blk=0) -> DeviceTensor4D:
    """Convolution and the max pooling that consumes it as one kernel
    (lcnn_conv_maxpool_packed): the pooled CHWN tensor, bit-identical to
    conv_forward_packed followed by pool_layout (max)."""
    torch = _torch()
    ho, wo = conv_output_extents(x.h, x.w, f_h, f_w, stride, pad)
    hp, wp = (ho - pool_win) // pool_stride + 1, (wo - pool_win) // pool_stride + 1
    if out is None:
        out = DeviceTensor4D(x.n, c_o, hp, wp, x.layout,
                             torch.empty(x.n * c_o * hp * wp, dtype=torch.float32,
                                         device=x.data.device))
    capi.call("lcnn_conv_maxpool_packed_blk", x.ptr(), packed.data_ptr(), out.ptr(), x.n, x.c,
              x.h, x.w, x.layout, c_o, f_h, f_w, stride, pad, precision, pool_win, pool_stride,
              blk, _stream(stream))
    return out


def gemm(a, b, m, n, k, precision=FP32, out=None, workspace=None, stream=None):
    """c (m x n) = a (m x k) * b (k x n), row-major fp32 CUDA tensors
    (gemm_blocked conv.cpp:252-304 / fc_forward softmax.cpp:182-184)."""
    torch = _torch()
    if out is None:
        out = torch.empty(m * n, dtype=torch.float32, device=a.device)
    nbytes = capi.lib().lcnn_gemm_workspace_bytes(m, n, k, precision)
    if workspace is None or workspace.numel() * 4 < nbytes:
        workspace = torch.empty(max(1, (nbytes + 3) // 4), dtype=torch.float32, device=a.device)
    capi.call("lcnn_gemm", a.data_ptr(), b.data_ptr(), out.data_ptr(), m, n, k, precision,
              workspace.data_ptr(), workspace.numel() * 4, _stream(stream))
    return out


def pack_fc_weights(weights, k, n, precision=TF32, stream=None):
    """fc weights (k x n row-major CUDA tensor) packed once into the
    tensor-core operand image (lcnn_fc_pack_weights) -> CUDA uint8 tensor."""
    torch = _torch()
    nbytes = capi.lib().lcnn_fc_packed_bytes(k, n, precision)
    if nbytes == 0:
        raise ValueError("fc: packed weights need TF32 or 3xTF32 precision")
    packed = torch.empty(nbytes, dtype=torch.uint8, device=weights.device)
    capi.call("lcnn_fc_pack_weights", weights.data_ptr(), packed.data_ptr(), nbytes, k, n,
              precision, _stream(stream))
    return packed


def fc_forward_packed(x, x_layout, packed, m, n, k, precision=TF32, out=None, stream=None,
                      sync=None, next_packed=None):
    """y (m x n) = x . W on packed weights.  x_layout NCHW: x is m rows of k;
    CHWN: x is [k][m] (a CHWN producer, flattened in the operand load).
    sync: optional zeroed CUDA tensor of >= capi.SYNC_BYTES bytes owned by this
    call site (lcnn_fc_forward_packed_ex: in-kernel stream-K zeroing).
    next_packed: the next fc layer's packed weights, prefetched into L2 by the
    CTAs of this one once their own loads are issued."""
    torch = _torch()
    if out is None:
        out = torch.empty(m * n, dtype=torch.float32, device=x.device)
    nbytes = capi.lib().lcnn_fc_workspace_bytes(m, k, precision)
    ws = torch.empty(max(1, (nbytes + 3) // 4), dtype=torch.float32, device=x.device)
    capi.call("lcnn_fc_forward_packed_ex", x.data_ptr(), x_layout, packed.data_ptr(),
              out.data_ptr(), m, n, k, precision, ws.data_ptr(), ws.numel() * 4,
              sync.data_ptr() if sync is not None else None,
              next_packed.data_ptr() if next_packed is not None else None,
              next_packed.numel() * next_packed.element_size() if next_packed is not None else 0,
              _stream(stream))
    return out


__all__ = ["TF32", "X3TF32", "FP32", "conv_forward", "gemm", "pack_conv_filters",
    "pack_fc_weights", "fc_forward_packed",
    "conv_forward_packed", "conv_maxpool_supported", "conv_maxpool_packed", "conv_output_extents",
    "NCHW", "CHWN", "NHWC", "HWCN", "MAX", "AVERAGE", "DeviceTensor4D", "DeviceMatrix",
    "TransformPlan", "PoolParams", "CoarseningPlan", "AccessReport", "PassReport",
    "flattenable_pair", "make_plan", "transform", "transform_tiled", "transform_naive",
    "pool_output_extents", "pool_layout", "pool_coarsened", "pool_coarsened_nchw",
    "pool_oracle", "softmax_fused", "softmax_reference", "layout_strides", "K_COARSENING_CAP",
    "field",
]
