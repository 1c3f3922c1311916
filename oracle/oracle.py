"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front-end of the CPU oracle.

Two CPU implementations of the reference algorithms, both used purely as
checkers (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline and
--impl reference legs):

* ``C``   -- oracle/build/liblcnn_oracle.so, the plain-C restatement in
             oracle/lcnn_oracle.c (each function cites reference file:line);
* ``Ref`` -- oracle/_ref/liblcnn_ref.so, the unmodified reference sources
             compiled by oracle/Makefile (+ ref_shim.cpp).  Absent on a box that
             never had /root/reference unless the prebuilt file travelled.

Arrays are flat float32 numpy buffers in the layout's memory order.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import CFUNCTYPE, POINTER, c_char_p, c_double, c_int, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB = os.path.join(HERE, "build", "liblcnn_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "liblcnn_ref.so")  # x86-64-v2 build (always present)


def _cpu_flags() -> set:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def ref_lib_path() -> tuple[str, str]:
    """(path, ISA level) of the highest reference build this CPU runs: the
    reference's own build is -march=native, so the CPU baseline
    is not handicapped by the generic build (oracle/Makefile)."""
    flags = _cpu_flags()
    v3 = {"avx2", "fma", "bmi1", "bmi2", "f16c", "movbe"}
    v4 = {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"}
    for level, need in (("x86-64-v4", v3 | v4), ("x86-64-v3", v3)):
        path = os.path.join(HERE, "_ref", f"liblcnn_ref_{level[-2:]}.so")
        if need <= flags and os.path.exists(path):
            return path, level
    return REF_LIB, "x86-64-v2"

NCHW, CHWN, NHWC, HWCN = 0, 1, 2, 3

COST_FN = CFUNCTYPE(c_double, c_uint32, c_uint32, c_void_p)
BENCH_FN = CFUNCTYPE(c_double, c_int, c_uint32, c_uint32, c_void_p)


class OracleError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _p(a):
    return a.ctypes.data_as(c_void_p)


def build_c() -> None:
    if not os.path.exists(C_LIB):
        subprocess.run(["make", "-C", HERE, "build/liblcnn_oracle.so"], check=True,
                       stdout=subprocess.DEVNULL)


class C:
    """The C restatement (oracle/lcnn_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            build_c()
            cls._lib = ctypes.CDLL(C_LIB)
        return cls._lib

    @classmethod
    def _rc(cls, rc, what):
        if rc:
            raise OracleError(rc, what)

    @classmethod
    def transform(cls, src, n, c, h, w, sl, dl):
        src = _f32(src)
        out = np.empty_like(src)
        cls._rc(cls.lib().orc_transform(_p(src), _p(out), n, c, h, w, sl, dl), "transform")
        return out

    @classmethod
    def pool_extents(cls, h, w, wh, ww, s):
        ho, wo = c_uint32(), c_uint32()
        cls._rc(cls.lib().orc_pool_extents(h, w, wh, ww, s, ctypes.byref(ho), ctypes.byref(wo)),
                "pool: window")
        return ho.value, wo.value

    @classmethod
    def pool_oracle(cls, src, n, c, h, w, layout, wh, ww, s, avg):
        ho, wo = cls.pool_extents(h, w, wh, ww, s)
        src = _f32(src)
        out = np.empty(n * c * ho * wo, np.float32)
        cls._rc(cls.lib().orc_pool_oracle(_p(src), _p(out), n, c, h, w, layout, wh, ww, s,
                                          int(avg)), "pool_oracle")
        return out

    @classmethod
    def pool_plain(cls, src, n, c, h, w, layout, wh, ww, s, avg):
        ho, wo = cls.pool_extents(h, w, wh, ww, s)
        src = _f32(src)
        out = np.empty(n * c * ho * wo, np.float32)
        rep = (c_uint64 * 3)()
        cls._rc(cls.lib().orc_pool_plain(_p(src), _p(out), n, c, h, w, layout, wh, ww, s,
                                         int(avg), rep), "pool_plain")
        return out, tuple(rep)

    @classmethod
    def pool_coarsened(cls, src, n, c, h, w, layout, wh, ww, s, avg, fh, fw):
        ho, wo = cls.pool_extents(h, w, wh, ww, s)
        src = _f32(src)
        out = np.empty(n * c * ho * wo, np.float32)
        rep = (c_uint64 * 3)()
        cls._rc(cls.lib().orc_pool_coarsened(_p(src), _p(out), n, c, h, w, layout, wh, ww, s,
                                             int(avg), fh, fw, rep), "pool_coarsened")
        return out, tuple(rep)

    @classmethod
    def softmax_reference(cls, x, rows, cols):
        x = _f32(x)
        out = np.empty_like(x)
        rep = (c_uint32 * 2)()
        cls._rc(cls.lib().orc_softmax_reference(_p(x), _p(out), rows, cols, rep), "softmax")
        return out, tuple(rep)

    @classmethod
    def softmax_fused(cls, x, rows, cols, limit=16384):
        x = _f32(x)
        out = np.empty_like(x)
        rep = (c_uint32 * 2)()
        cls._rc(cls.lib().orc_softmax_fused(_p(x), _p(out), rows, cols, limit, rep), "softmax")
        return out, tuple(rep)

    @classmethod
    def conv_extents(cls, h, w, fh, fw, stride, pad):
        ho, wo = c_uint32(), c_uint32()
        cls._rc(cls.lib().orc_conv_extents(h, w, fh, fw, stride, pad, ctypes.byref(ho),
                                           ctypes.byref(wo)), "conv extents")
        return ho.value, wo.value

    @classmethod
    def conv_oracle(cls, x, filt, n, ci, h, w, layout, co, fh, fw, stride, pad):
        ho, wo = cls.conv_extents(h, w, fh, fw, stride, pad)
        x, filt = _f32(x), _f32(filt)
        out = np.empty(n * co * ho * wo, np.float32)
        cls._rc(cls.lib().orc_conv_oracle(_p(x), _p(filt), _p(out), n, ci, h, w, layout, co, fh,
                                          fw, stride, pad), "conv_oracle")
        return out

    @classmethod
    def gemm(cls, a, b, m, n, k):
        a, b = _f32(a), _f32(b)
        out = np.empty(m * n, np.float32)
        cls.lib().orc_gemm_f64(_p(a), _p(b), _p(out), c_uint64(m), c_uint64(n), c_uint64(k))
        return out

    @classmethod
    def choose_layout(cls, kind, n, c, c_t, n_t):
        return cls.lib().orc_choose_layout(kind, n, c, c_t, n_t)

    @classmethod
    def calibrate(cls, bench):
        cb = BENCH_FN(lambda l, n, c, ctx: bench(l, n, c))
        ct, nt = c_uint32(), c_uint32()
        cls.lib().orc_calibrate(cb, None, ctypes.byref(ct), ctypes.byref(nt))
        return ct.value, nt.value

    @classmethod
    def autotune(cls, cost):
        cb = COST_FN(lambda fh, fw, ctx: cost(fh, fw))
        fh, fw = c_uint32(), c_uint32()
        cls.lib().orc_autotune(cb, None, ctypes.byref(fh), ctypes.byref(fw))
        return fh.value, fw.value

    @classmethod
    def plan_transforms(cls, kinds, layouts):
        k = (c_int * len(kinds))(*kinds)
        l = (c_int * len(layouts))(*layouts)
        pos, src, dst = (c_int * 64)(), (c_int * 64)(), (c_int * 64)()
        cnt = cls.lib().orc_plan_transforms(k, l, len(kinds), pos, src, dst)
        return [(pos[i], src[i], dst[i]) for i in range(cnt)]


class Ref:
    """The unmodified reference library (oracle/_ref/liblcnn_ref.so)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_LIB)

    @classmethod
    def variant(cls) -> str:
        """'-O2 -march=<level>' of the build Ref.lib() loads."""
        return f"g++ -O2 -march={ref_lib_path()[1]} ({os.path.basename(ref_lib_path()[0])})"

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not cls.available():
                raise FileNotFoundError(REF_LIB)
            dll = ctypes.CDLL(ref_lib_path()[0])
            dll.ref_last_error.restype = c_char_p
            dll.ref_session_create.restype = c_void_p
            dll.ref_session_create.argtypes = [c_int] + [c_uint32] * 4 + [c_int, c_int] + \
                [c_uint32] * 3 + [c_int] + [c_uint32] * 2 + [c_int]
            dll.ref_session_run.restype = c_double
            dll.ref_session_run.argtypes = [c_void_p]
            dll.ref_session_destroy.argtypes = [c_void_p]
            dll.ref_gemm_blocked.argtypes = [c_void_p] * 3 + [c_uint64] * 3
            dll.ref_time_network.restype = c_double
            dll.ref_time_network.argtypes = [c_char_p, c_uint32, c_uint32, c_int]
            cls._lib = dll
        return cls._lib

    @classmethod
    def _rc(cls, rc):
        if rc:
            raise OracleError(rc, cls.lib().ref_last_error().decode())

    @classmethod
    def transform(cls, src, n, c, h, w, sl, dl):
        src = _f32(src)
        out = np.empty_like(src)
        cls._rc(cls.lib().ref_transform(_p(src), _p(out), n, c, h, w, sl, dl))
        return out

    @classmethod
    def transform_tiled(cls, src, n, c, h, w, sl, dl, tile=32, wide=False):
        src = _f32(src)
        out = np.empty_like(src)
        cls._rc(cls.lib().ref_transform_tiled(_p(src), _p(out), n, c, h, w, sl, dl, tile,
                                              int(wide)))
        return out

    @classmethod
    def pool_oracle(cls, src, n, c, h, w, layout, wh, ww, s, avg):
        ho, wo = (h - wh) // s + 1, (w - ww) // s + 1
        src = _f32(src)
        out = np.empty(n * c * ho * wo, np.float32)
        cls._rc(cls.lib().ref_pool_oracle(_p(src), _p(out), n, c, h, w, layout, wh, ww, s,
                                          int(avg)))
        return out

    @classmethod
    def pool_layout(cls, src, n, c, h, w, layout, wh, ww, s, avg):
        ho, wo = (h - wh) // s + 1, (w - ww) // s + 1
        src = _f32(src)
        out = np.empty(n * c * ho * wo, np.float32)
        rep = (c_uint64 * 3)()
        cls._rc(cls.lib().ref_pool_layout(_p(src), _p(out), n, c, h, w, layout, wh, ww, s,
                                          int(avg), rep))
        return out, tuple(rep)

    @classmethod
    def pool_coarsened(cls, src, n, c, h, w, layout, wh, ww, s, avg, fh, fw):
        ho, wo = (h - wh) // s + 1, (w - ww) // s + 1
        src = _f32(src)
        out = np.empty(n * c * ho * wo, np.float32)
        rep = (c_uint64 * 3)()
        cls._rc(cls.lib().ref_pool_coarsened(_p(src), _p(out), n, c, h, w, layout, wh, ww, s,
                                             int(avg), fh, fw, rep))
        return out, tuple(rep)

    @classmethod
    def softmax_reference(cls, x, rows, cols):
        x = _f32(x)
        out = np.empty_like(x)
        rep = (c_uint32 * 2)()
        cls._rc(cls.lib().ref_softmax_reference(_p(x), _p(out), rows, cols, rep))
        return out, tuple(rep)

    @classmethod
    def softmax_fused(cls, x, rows, cols, limit=16384):
        x = _f32(x)
        out = np.empty_like(x)
        rep = (c_uint32 * 2)()
        cls._rc(cls.lib().ref_softmax_fused(_p(x), _p(out), rows, cols, limit, rep))
        return out, tuple(rep)

    @classmethod
    def conv_oracle(cls, x, filt, n, ci, h, w, layout, co, fh, fw, stride, pad):
        ho = (h + 2 * pad - fh) // stride + 1
        wo = (w + 2 * pad - fw) // stride + 1
        x, filt = _f32(x), _f32(filt)
        out = np.empty(n * co * ho * wo, np.float32)
        cls._rc(cls.lib().ref_conv_oracle(_p(x), _p(filt), _p(out), n, ci, h, w, layout, co, fh,
                                          fw, stride, pad))
        return out

    @classmethod
    def conv_direct(cls, x, filt, n, ci, h, w, layout, co, fh, fw, stride, pad):
        ho = (h + 2 * pad - fh) // stride + 1
        wo = (w + 2 * pad - fw) // stride + 1
        x, filt = _f32(x), _f32(filt)
        out = np.empty(n * co * ho * wo, np.float32)
        cls._rc(cls.lib().ref_conv_direct(_p(x), _p(filt), _p(out), n, ci, h, w, layout, co, fh,
                                          fw, stride, pad))
        return out

    @classmethod
    def gemm_blocked(cls, a, b, m, n, k):
        a, b = _f32(a), _f32(b)
        out = np.empty(m * n, np.float32)
        cls._rc(cls.lib().ref_gemm_blocked(_p(a), _p(b), _p(out), m, n, k))
        return out

    @classmethod
    def choose_layout(cls, kind, n, c, c_t, n_t):
        return cls.lib().ref_choose_layout(kind, n, c, c_t, n_t)

    @classmethod
    def calibrate(cls, bench):
        cb = BENCH_FN(lambda l, n, c, ctx: bench(l, n, c))
        ct, nt = c_uint32(), c_uint32()
        cls._rc(cls.lib().ref_calibrate(cb, None, ctypes.byref(ct), ctypes.byref(nt)))
        return ct.value, nt.value

    @classmethod
    def autotune(cls, cost, dims=(4, 4, 24, 24), params=(3, 3, 2, 0)):
        cb = COST_FN(lambda fh, fw, ctx: cost(fh, fw))
        fh, fw = c_uint32(), c_uint32()
        cls._rc(cls.lib().ref_autotune_pool(*dims, *params, cb, None, ctypes.byref(fh),
                                            ctypes.byref(fw)))
        return fh.value, fw.value

    @classmethod
    def plan_network(cls, json_text, c_t=0, n_t=0):
        layouts = (c_int * 64)()
        steps = c_int()
        pos, src, dst = (c_int * 64)(), (c_int * 64)(), (c_int * 64)()
        cls._rc(cls.lib().ref_plan_network(json_text.encode(), c_t, n_t, layouts, 64,
                                           ctypes.byref(steps), pos, src, dst, 64))
        return list(layouts), [(pos[i], src[i], dst[i]) for i in range(steps.value)]

    @classmethod
    def run_network(cls, json_text, x, in_layout, c_t=0, n_t=0, seed=42, out_cap=1 << 24):
        """The unmodified run_network on input x (flat, in in_layout) ->
        (rows, cols) float32 matrix (ref_shim.cpp ref_run_network)."""
        x = _f32(x)
        out = np.empty(out_cap, np.float32)
        rows, cols = c_uint32(), c_uint32()
        cls._rc(cls.lib().ref_run_network(json_text.encode(), c_t, n_t, c_uint64(seed), _p(x),
                                          in_layout, _p(out), c_uint64(out_cap),
                                          ctypes.byref(rows), ctypes.byref(cols)))
        return out[:rows.value * cols.value].reshape(rows.value, cols.value).copy()

    @classmethod
    def run_network_sharded(cls, json_text, x, n, c_t=0, n_t=0, seed=42, threads=None,
                            out_cap=1 << 26):
        """ref_run_network_sharded: the unmodified run_network on NCHW input x
        (n images), N-sharded over host threads (each shard annotated with its
        own per-shard n) -> (n, cols) float32."""
        x = _f32(x)
        threads = threads or len(os.sched_getaffinity(0))
        out = np.empty(out_cap, np.float32)
        rows, cols = c_uint32(), c_uint32()
        cls._rc(cls.lib().ref_run_network_sharded(json_text.encode(), c_t, n_t, c_uint64(seed),
                                                  _p(x), n, _p(out), c_uint64(out_cap),
                                                  ctypes.byref(rows), ctypes.byref(cols),
                                                  threads))
        return out[:rows.value * cols.value].reshape(rows.value, cols.value).copy()

    @classmethod
    def session(cls, op, n, c, h, w, layout=NCHW, dst_layout=NCHW, wh=1, ww=1, s=1, avg=False,
                fh=1, fw=1, threads=1):
        """A timed reference call over an n-image batch split into `threads`
        N-shards (ref_shim.cpp ref_session_*); inputs are built once."""
        return RefSession(cls.lib(), op, n, c, h, w, layout, dst_layout, wh, ww, s, avg, fh, fw,
                          threads)


def ref_time_network(json_text: str, c_t: int, n_t: int, threads: int) -> float:
    """Seconds of the reference run_network with `threads` concurrent shards
    (each shard's batch is the config's n)."""
    t = Ref.lib().ref_time_network(json_text.encode(), c_t, n_t, threads)
    if t < 0:
        raise OracleError(11, Ref.lib().ref_last_error().decode())
    return t


class RefSession:
    def __init__(self, lib, *args):
        self._lib = lib
        self._h = lib.ref_session_create(*[int(a) for a in args])
        if not self._h:
            raise OracleError(11, lib.ref_last_error().decode())

    def run(self) -> float:
        t = self._lib.ref_session_run(self._h)
        if t < 0:
            raise OracleError(11, self._lib.ref_last_error().decode())
        return t

    def close(self):
        if self._h:
            self._lib.ref_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


OP_POOL_LAYOUT, OP_POOL_COARSENED, OP_SOFTMAX_FUSED, OP_SOFTMAX_REFERENCE, OP_TRANSFORM, \
    OP_TRANSFORM_NAIVE = range(6)


def rng_uniform(seed, size, lo=-1.0, hi=1.0):
    """Seeded fp32 uniform input (the reference's tests use mt19937 +
    uniform_real_distribution; parity only needs identical inputs on both
    sides, so a numpy generator is used)."""
    return np.random.default_rng(seed).uniform(lo, hi, size).astype(np.float32)


def approx_equal(a, b, rel_tol) -> bool:
    """== approx_equal (tensor.cpp:157-187) on same-order flat buffers."""
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), np.float32(1.0))
    diff = np.abs(a - b)
    return not bool(np.any(diff > np.float32(rel_tol) * scale))


def bit_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


__all__ = ["C", "Ref", "OracleError", "approx_equal", "bit_equal", "rng_uniform", "NCHW", "CHWN",
           "NHWC", "HWCN", "POINTER"]
