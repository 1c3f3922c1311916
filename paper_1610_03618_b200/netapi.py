"""ctypes binding of the network runtime C ABI (include/lcnn_net.h, in
lib/liblcnn.so): parse + annotate + upload weights once, then device-resident
(or host-buffer) forward passes."""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_int, c_uint32, c_uint64, c_void_p

from .capi import PKG_DIR, PoolPlan
from .errors import raise_for_status

LIB = os.path.join(PKG_DIR, "lib", "liblcnn.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run make / __graft_entry__.build()")
        d = ctypes.CDLL(LIB)
        d.lcnn_net_create.argtypes = [c_char_p, c_uint32, c_uint32, c_uint64, POINTER(c_void_p)]
        d.lcnn_net_create_ex.argtypes = [c_char_p, c_uint32, c_uint32, c_uint64, c_int,
                                         POINTER(c_void_p)]
        d.lcnn_net_precision.argtypes = [c_void_p]
        d.lcnn_net_pool_plan.argtypes = [c_void_p, c_uint32, POINTER(PoolPlan)]
        d.lcnn_net_status.argtypes = [c_void_p, c_void_p]
        d.lcnn_net_nonfinite_flag.argtypes = [c_void_p]
        d.lcnn_net_nonfinite_flag.restype = c_void_p
        d.lcnn_net_destroy.argtypes = [c_void_p]
        d.lcnn_net_last_error.restype = c_char_p
        d.lcnn_net_info.argtypes = [c_void_p, c_int, POINTER(c_uint32), POINTER(c_int),
                                    POINTER(c_uint32), POINTER(c_uint32), POINTER(c_uint64),
                                    POINTER(c_uint32)]
        d.lcnn_net_layouts.argtypes = [c_void_p, POINTER(c_int), c_uint32]
        d.lcnn_net_forward.argtypes = [c_void_p, c_void_p, c_int, c_void_p, c_void_p]
        d.lcnn_net_forward_graph.argtypes = [c_void_p, c_void_p, c_int, c_void_p, c_void_p]
        d.lcnn_net_forward_host.argtypes = [c_void_p, c_void_p, c_int, c_void_p]
        d.lcnn_net_forward_host_many.argtypes = [c_void_p, POINTER(c_void_p), c_int,
                                                 POINTER(c_void_p), c_uint32]
        d.lcnn_set_dense_precision.argtypes = [c_int]
        d.lcnn_net_profile.argtypes = [c_void_p, c_void_p, c_int, c_void_p, POINTER(c_uint64),
                                       c_uint32, c_char_p, ctypes.c_size_t, POINTER(c_uint32)]
        _lib = d
    return _lib


def _check(st):
    if st:
        raise_for_status(st, lib().lcnn_net_last_error().decode())


class Network:
    """A parsed, annotated network with weights resident in HBM."""

    def __init__(self, json_text: str, c_t: int = 0, n_t: int = 0, seed: int = 42,
                 precision: int | None = None):
        """precision: capi.PREC_* for the conv / fc layers (None = the process
        default set by set_dense_precision)."""
        h = c_void_p()
        _check(lib().lcnn_net_create_ex(json_text.encode(), c_t, n_t, seed,
                                        -1 if precision is None else precision,
                                        ctypes.byref(h)))
        self._h = h
        self.layouts = self._layouts()
        self.precision = lib().lcnn_net_precision(self._h)

    def info(self, in_layout: int):
        dims = (c_uint32 * 4)()
        first, rows, cols, flops, tr = c_int(), c_uint32(), c_uint32(), c_uint64(), c_uint32()
        _check(lib().lcnn_net_info(self._h, in_layout, dims, ctypes.byref(first),
                                   ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(flops),
                                   ctypes.byref(tr)))
        return {"dims": tuple(dims), "first_layout": first.value, "out": (rows.value, cols.value),
                "flops_per_image": flops.value, "transforms": tr.value}

    def _layouts(self):
        arr = (c_int * 256)()
        _check(lib().lcnn_net_layouts(self._h, arr, 256))
        return list(arr)

    def forward(self, d_input: int, in_layout: int, d_output: int, stream: int):
        _check(lib().lcnn_net_forward(self._h, d_input, in_layout, d_output, stream))

    def forward_graph(self, d_input: int, in_layout: int, d_output: int, stream: int):
        """lcnn_net_forward_graph: the forward replayed from a CUDA graph the
        network captures once per (input, layout, output) buffer triple."""
        _check(lib().lcnn_net_forward_graph(self._h, d_input, in_layout, d_output, stream))

    def pool_plans(self):
        """{layer index: PoolPlan} of the network's pooling layers (tuned at creation)."""
        out = {}
        for i in range(len(self.layouts)):
            p = PoolPlan()
            if lib().lcnn_net_pool_plan(self._h, i, ctypes.byref(p)) == 0 and p.tuned:
                out[i] = p
        return out

    def status(self, stream: int):
        """Wait for `stream`; raise DomainError if a forward since the last
        call met a non-finite classifier input (clears the flag)."""
        _check(lib().lcnn_net_status(self._h, stream))

    def nonfinite_flag_ptr(self) -> int:
        """Device address of the sticky non-finite flag (an int32)."""
        return lib().lcnn_net_nonfinite_flag(self._h)

    def forward_host(self, h_input: int, in_layout: int, h_output: int):
        _check(lib().lcnn_net_forward_host(self._h, h_input, in_layout, h_output))

    def forward_host_many(self, h_inputs, in_layout: int, h_outputs):
        """Pipelined forwards over host buffers (pointer lists of equal length):
        batch i+1's H2D overlaps batch i's forward."""
        if len(h_inputs) != len(h_outputs):
            raise ValueError("h_inputs and h_outputs differ in length")
        n = len(h_inputs)
        ins = (c_void_p * max(n, 1))(*h_inputs)
        outs = (c_void_p * max(n, 1))(*h_outputs)
        _check(lib().lcnn_net_forward_host_many(self._h, ins, in_layout, outs, n))

    def profile(self, d_input: int, in_layout: int, stream: int):
        """[(entry name, device nanoseconds)] of one forward."""
        nanos = (c_uint64 * 256)()
        names = ctypes.create_string_buffer(8192)
        count = c_uint32()
        _check(lib().lcnn_net_profile(self._h, d_input, in_layout, stream, nanos, 256, names,
                                      8192, ctypes.byref(count)))
        labels = names.value.decode().split(",") if count.value else []
        return list(zip(labels, [nanos[i] for i in range(count.value)]))

    def close(self):
        if getattr(self, "_h", None):
            lib().lcnn_net_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def set_dense_precision(precision: int) -> None:
    lib().lcnn_set_dense_precision(precision)
