#!/usr/bin/env python
"""Benchmark of the B200 memory-bound CNN layer path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload vgg_pools|pl5|pl5_nchw|softmax|softmax5|transform]

A *step* is one pass of the hot path over one batch of synthetic input that
is already resident in HBM.  The default workload is BASELINE config 4: the
five VGG-16 pooling layers (max 2x2/s2) on a 256-image batch per GPU in CHWN,
the layout the paper's selector assigns to pooling.  Batch N shards across
GPUs with no collective on the data path (weak scaling: 256 images per GPU);
NCCL is used only for the timing barrier and the max-over-ranks reduction.

Rank 0 prints ONE JSON line carrying the contract keys plus `roofline`
(dominant kernel: achieved algorithmic GB/s vs the measured HBM copy peak),
`cpu_baseline` (the reference CPU path timed on this host's cores), `e2e`
(host buffers: pinned H2D + kernel + D2H in the timed region), `clocks` and
`gpu_launches`.  `--impl reference` times the unmodified reference library
(oracle/_ref) on the same workload's per-step sample with all host cores.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Layer GB/s vs HBM peak (pool/softmax/transpose); AlexNet fwd images/sec"
GB = 1e9

# BASELINE config 4: VGG-16 pooling inputs (C, H) with H == W, max 2x2 stride 2
VGG_POOLS = [(64, 224), (128, 112), (256, 56), (512, 28), (512, 14)]
# BASELINE config 3: AlexNet (fixture-consistent) + VGG-16 activations (C, H, W)
TRANSFORM_SHAPES = [(3, 227, 227), (96, 55, 55), (96, 27, 27), (192, 27, 27), (192, 13, 13),
                    (384, 13, 13), (256, 13, 13), (256, 6, 6), (3, 224, 224), (64, 224, 224),
                    (64, 112, 112), (128, 112, 112), (128, 56, 56), (256, 56, 56), (256, 28, 28),
                    (512, 28, 28), (512, 14, 14), (512, 7, 7)]


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from the committed ncu --set full summary (profiles/)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# ------------------------------------------------------------------ ops ----
# An Op is constructed from SHAPES ONLY (no torch, no CUDA library): the
# reference arm describes and runs the same workload from these objects
# without ever loading paper_1610_03618_b200.  alloc() binds device buffers
# and the C ABI for our arm.
L2_BYTES = 126 << 20  # B200 L2 (cudaDevAttrL2CacheSize 126.5 MiB), rounded down
LAYOUT_NAMES = {0: "nchw", 1: "chwn", 2: "nhwc", 3: "hwcn"}


def l2_rotations(footprint):
    """Input/output copies a single-op workload rotates over so that no
    buffer is re-read from L2: enough to stream > 4x L2 between reuses when
    one launch touches less than 2x L2 (SURVEY 8d timing method)."""
    return max(1, min(16, -(-4 * L2_BYTES // footprint))) if footprint < 2 * L2_BYTES else 1


class Op:
    """One launch of a hot-path kernel on device-resident buffers."""

    name = "op"
    in_bytes = 0
    out_bytes = 0
    rot = 1  # rotated input/output copies (single-op workloads smaller than 2x L2)
    _i = 0   # launches so far (selects the copy)
    _args = None

    @property
    def bytes(self):
        return self.in_bytes + self.out_bytes

    @property
    def units(self):
        """Images (rows for softmax) one launch processes."""
        return getattr(self, "n", None) or getattr(self, "rows")

    def next_views(self):
        """The (input, output) slices the next launch() will use."""
        r = self._i % self.rot
        nx, ny = self.in_bytes // 4, self.out_bytes // 4
        return self.x[r * nx:(r + 1) * nx], self.y[r * ny:(r + 1) * ny]

    def alloc(self, torch, device):
        from paper_1610_03618_b200 import capi

        self.capi, self.lib = capi, capi.lib()
        g = torch.Generator(device=device).manual_seed(self.seed)
        lo, hi = self.data_range
        self.x = torch.rand(self.rot * self.in_bytes // 4, device=device, generator=g) * (hi - lo) + lo
        self.y = torch.empty(self.rot * self.out_bytes // 4, device=device)
        self._extra_alloc(torch, device)
        self._args = [self.bind(self.x.data_ptr() + r * self.in_bytes,
                                self.y.data_ptr() + r * self.out_bytes) for r in range(self.rot)]
        return self

    data_range = (-1.0, 1.0)

    def _extra_alloc(self, torch, device):
        pass

    def launch(self, stream):
        fn, args = self._args[self._i % self.rot]
        self._i += 1
        st = fn(*args, stream)
        if st:
            self.capi.check(st, self.name)

    def ref_session(self, batch, threads):
        raise NotImplementedError


class PoolOp(Op):
    def __init__(self, n, c, h, w, layout, win, stride, avg, plan, seed, rotate=False):
        self.n, self.c, self.h, self.w = n, c, h, w
        self.layout, self.win, self.stride, self.avg = layout, win, stride, avg
        self.plan = plan  # None = the GPU-tuned plan (lcnn_pool_tune at alloc)
        self.seed = seed
        self.ho = (h - win) // stride + 1
        self.wo = (w - win) // stride + 1
        self.in_bytes = n * c * h * w * 4
        self.out_bytes = n * c * self.ho * self.wo * 4
        self.rot = l2_rotations(self.in_bytes + self.out_bytes) if rotate else 1
        kind = "plain" if plan is None else f"coarsened({plan[0]},{plan[1]})"
        self.name = f"pool_{LAYOUT_NAMES[layout]}_{kind}_{n}x{c}x{h}x{w}_w{win}s{stride}"

    def _extra_alloc(self, torch, device):
        self.rep = self.capi.AccessReport()
        if self.plan is None:
            # the GPU autotuner (lcnn_pool_tune): every specialised kernel plan
            # of this layout timed on this shape, fastest cached and used
            self.tuned = self.capi.PoolPlan()
            st = self.lib.lcnn_pool_tune(self.n, self.c, self.h, self.w, self.layout, self.win,
                                         self.win, self.stride, 1 if self.avg else 0,
                                         ctypes.byref(self.tuned),
                                         torch.cuda.current_stream(device).cuda_stream)
            self.capi.check(st, "pool_tune")
            t = self.tuned
            ring = f",ring{t.ring_kb}KBx{t.ring_slots}x{t.ring_ctas}" if t.ring_kb else ""
            self.name = self.name.replace("_plain_", f"_tuned({t.fh},{t.fw}{ring})_")

    def bind(self, x_ptr, y_ptr):
        mode = 1 if self.avg else 0
        if self.plan is None:
            fn = self.lib.lcnn_pool_run_plan
            args = (x_ptr, y_ptr, self.n, self.c, self.h, self.w, self.layout, self.win, self.win,
                    self.stride, mode, ctypes.byref(self.tuned), ctypes.byref(self.rep))
        elif self.layout == 1:
            fn = self.lib.lcnn_pool_coarsened
            args = (x_ptr, y_ptr, self.n, self.c, self.h, self.w, self.layout, self.win, self.win,
                    self.stride, mode, self.plan[0], self.plan[1], ctypes.byref(self.rep))
        else:
            fn = self.lib.lcnn_pool_coarsened_nchw
            args = (x_ptr, y_ptr, self.n, self.c, self.h, self.w, self.win, self.win, self.stride,
                    mode, self.plan[0], self.plan[1], ctypes.byref(self.rep))
        return fn, args

    def ref_session(self, batch, threads):
        """The reference call for this layer: pool_coarsened for a CHWN plan,
        pool_layout otherwise (NCHW has no coarsened reference, pool.cpp:190)."""
        from oracle.oracle import OP_POOL_COARSENED, OP_POOL_LAYOUT, Ref

        # the reference's pool_layout (pool.cpp:172-176, its faster pooling
        # entry on both layouts: PL5 2.60 vs 2.30 GB/s for pool_coarsened(2,2));
        # an explicit CHWN --plan runs the reference's pool_coarsened
        op = OP_POOL_COARSENED if self.plan and self.layout == 1 else OP_POOL_LAYOUT
        fh, fw = self.plan or (1, 1)
        s = Ref.session(op, batch, self.c, self.h, self.w, self.layout, 0, self.win, self.win,
                        self.stride, self.avg, fh, fw, threads)
        sample_bytes = batch * (self.c * self.h * self.w + self.c * self.ho * self.wo) * 4
        return s, sample_bytes


class SoftmaxOp(Op):
    data_range = (-5.0, 5.0)

    def __init__(self, rows, cols, fused, seed):
        self.rows, self.cols, self.fused, self.seed = rows, cols, fused, seed
        # bench.cpp:151 -- both arms are charged 2*N*C*4 algorithmic bytes
        self.in_bytes = self.out_bytes = rows * cols * 4
        # L2 policy: a matrix pair smaller than the 126 MB L2 would stay
        # resident between launches, so consecutive launches rotate over
        # enough (input, output) pairs to stream > 4x L2
        self.rot = l2_rotations(self.bytes)
        self.name = f"softmax_{'fused' if fused else 'five_pass'}_{rows}x{cols}"

    def _extra_alloc(self, torch, device):
        nbytes = self.lib.lcnn_softmax_reference_scratch_bytes(self.rows, self.cols)
        self.scratch = None if self.fused else torch.empty(nbytes // 4, device=device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)

    def bind(self, x_ptr, y_ptr):
        if self.fused:
            # the classifier form the network executor runs: one kernel per
            # step, the non-finite test ORed into a device flag that is never
            # re-zeroed (lcnn_softmax_fused zeroes its flag with an extra launch)
            return self.lib.lcnn_softmax_fused_sticky, (x_ptr, y_ptr, self.rows, self.cols,
                                                        self.flag.data_ptr())
        # the five-kernel baseline exactly (max, subtract, exp, sum, scale): no
        # flag, so no zeroing launch is charged to it either
        return self.lib.lcnn_softmax_reference, (x_ptr, y_ptr, self.rows, self.cols,
                                                 self.scratch.data_ptr(), self.scratch.numel() * 4,
                                                 None, None)

    def ref_session(self, batch, threads):
        from oracle.oracle import OP_SOFTMAX_FUSED, OP_SOFTMAX_REFERENCE, Ref

        op = OP_SOFTMAX_FUSED if self.fused else OP_SOFTMAX_REFERENCE
        s = Ref.session(op, batch, self.cols, 1, 1, 0, 0, 1, 1, 1, False, 1, 1, threads)
        return s, 2 * batch * self.cols * 4


class TransformOp(Op):
    data_range = (0.0, 1.0)

    def __init__(self, n, c, h, w, src, dst, seed, rotate=False):
        self.n, self.c, self.h, self.w, self.src, self.dst = n, c, h, w, src, dst
        self.seed = seed
        self.in_bytes = self.out_bytes = n * c * h * w * 4  # bench.cpp:202
        self.rot = l2_rotations(self.bytes) if rotate else 1
        self.name = (f"transform_{LAYOUT_NAMES[src]}_{LAYOUT_NAMES[dst]}_{n}x{c}x{h}x{w}")

    def bind(self, x_ptr, y_ptr):
        return self.lib.lcnn_transform, (x_ptr, y_ptr, self.n, self.c, self.h, self.w, self.src,
                                         self.dst)

    def ref_session(self, batch, threads):
        from oracle.oracle import OP_TRANSFORM, Ref

        s = Ref.session(OP_TRANSFORM, batch, self.c, self.h, self.w, self.src, self.dst, 1, 1, 1,
                        False, 1, 1, threads)
        return s, 2 * batch * self.c * self.h * self.w * 4


# ------------------------------------------------------------ workloads ----
class Workload:
    """What one rank runs (ops) plus the config dict both arms print.

    ops        -- this rank's launches per step (its N-shard for strong scaling)
    global_ops -- the whole job's ops on one device (what --impl reference runs)
    """

    def __init__(self, ops, global_ops, desc, dom, scaling, global_units, unit_name):
        self.ops, self.global_ops, self.desc, self.dom = ops, global_ops, desc, dom
        self.scaling, self.global_units, self.unit_name = scaling, global_units, unit_name

    @property
    def step_bytes_global(self):
        return sum(op.bytes for op in self.global_ops)


# BASELINE config 4's global batch.  LCNN_BENCH_VGG_GLOBAL overrides it for
# what-if runs (e.g. 32: one GPU's shard of an 8-GPU strong-scaled run); the
# config dict then reports the batch actually run.
VGG_GLOBAL_BATCH = int(os.environ.get("LCNN_BENCH_VGG_GLOBAL", "256"))


def build_workload(name, world, rank, plan=None, tsweep_n=None):
    """Shape-only description of a workload for `rank` of `world` GPUs.

    vgg_pools* is BASELINE config 4 as stated there: a GLOBAL batch of 256
    N-sharded over the GPUs (strong scaling, 256/G images per GPU).  The
    single-op configs (1-3) keep their per-GPU batch (weak scaling)."""
    from paper_1610_03618_b200.shard import shard_range  # pure python, no CUDA

    CHWN, NCHW = 1, 0
    seed = 1234 + 17 * rank
    par = f"N-shard x{world} (no data-path collective)"
    if name in ("vgg_pools", "vgg_pools_nchw"):
        layout = CHWN if name == "vgg_pools" else NCHW
        plans = [tuple(plan) if plan else None] * len(VGG_POOLS)  # None: GPU-tuned
        a, b = shard_range(VGG_GLOBAL_BATCH, world, rank)

        def mk(nb, sd):
            return [PoolOp(nb, c, hw, hw, layout, 2, 2, False, plans[i], sd + i)
                    for i, (c, hw) in enumerate(VGG_POOLS)]

        ops = mk(b - a, seed)
        gops = mk(VGG_GLOBAL_BATCH, 1234)
        lname = "CHWN (selector's pooling layout)" if layout == CHWN else "NCHW"
        gbytes = sum(op.bytes for op in gops)
        desc = {"workload": f"BASELINE config 4: VGG-16 pool1..pool5, max 2x2/s2, {lname}, "
                            f"global batch {VGG_GLOBAL_BATCH} N-sharded over {world} GPU(s)",
                "global_batch": VGG_GLOBAL_BATCH,
                "batch_per_gpu": [list(shard_range(VGG_GLOBAL_BATCH, world, r)) for r in range(world)]
                if world > 1 else VGG_GLOBAL_BATCH,
                "layers": [f"{VGG_GLOBAL_BATCH}x{c}x{hw}x{hw}" for c, hw in VGG_POOLS],
                "parallelism": par,
                "l2_policy": f"each step streams {gbytes / GB / world:.2f} GB per GPU "
                             "(>> 126 MB L2) between reuses of any buffer; no explicit flush"}
        return Workload(ops, gops, desc, 0, "strong", VGG_GLOBAL_BATCH, "images")
    if name in ("pl5", "pl5_nchw", "pl5_avg", "pl5_nchw_avg"):
        layout = CHWN if name in ("pl5", "pl5_avg") else NCHW
        avg = name.endswith("_avg")  # average pooling on the same shape (pool.cpp:98-134)
        p = tuple(plan) if plan else None  # None: GPU-tuned (lcnn_pool_tune)
        ops = [PoolOp(128, 96, 55, 55, layout, 3, 2, avg, p, seed, rotate=True)]
        desc = {"workload": f"BASELINE config 1: AlexNet pool1 (PL5) {'avg' if avg else 'max'} "
                            f"3x3/s2, 128x96x55x55, {'CHWN' if layout == CHWN else 'NCHW'}",
                "batch_per_gpu": 128, "global_batch": 128 * world, "parallelism": par,
                "l2_policy": f"{ops[0].rot} rotated input/output pairs "
                             f"({ops[0].rot * ops[0].bytes / 1e6:.0f} MB) between launches"}
        return Workload(ops, ops, desc, 0, "weak", 128 * world, "images")
    if name.startswith("softmax"):
        fused = not name.startswith("softmax5")
        rows, cols = 4096, 1000
        if name == "softmax_64k":
            rows = 65536
        elif name.endswith("_10k") or name.endswith("_10kcls"):
            # the paper's softmax comparison runs 10000 categories
            cols = 10000
        elif "_c" in name and name.rsplit("_c", 1)[-1].isdigit():
            cols = int(name.rsplit("_c", 1)[-1])  # softmax_cCOLS: 4096 rows of COLS
        elif "_" in name and name.split("_")[-1].isdigit():
            rows = int(name.split("_")[-1])
        ops = [SoftmaxOp(rows, cols, fused, seed)]
        desc = {"workload": f"BASELINE config 2: softmax classifier {rows}x{cols}, "
                            f"{'fused single kernel' if fused else 'five-kernel baseline'}"
                            + (" (HBM asymptote beyond the 4096-row config)" if rows > 4096 else "")
                            + (" (the paper's 10000-category case)" if cols != 1000 else ""),
                "batch_per_gpu": rows, "global_batch": rows * world, "parallelism": par,
                "l2_policy": (f"{ops[0].rot} rotated input/output pairs "
                              f"({ops[0].rot * ops[0].bytes / 1e6:.0f} MB > 4x L2) between launches"
                              if ops[0].rot > 1 else "matrix pair > 2x L2")}
        return Workload(ops, ops, desc, 0, "weak", rows * world, "rows")
    if name.startswith("transform"):
        # transform[_nchw|_nhwc|_hwcn][_N]: CHWN->NCHW (default), NCHW->CHWN,
        # or the generic permutations NCHW->NHWC / CHWN->HWCN (transform_naive) at batch N
        NHWC, HWCN = 2, 3
        src, dst = ((NCHW, CHWN) if "_nchw" in name else (NCHW, NHWC) if "_nhwc" in name
                    else (CHWN, HWCN) if "_hwcn" in name else (CHWN, NCHW))
        b = tsweep_n or 128
        if name.split("_")[-1].isdigit():
            b = int(name.split("_")[-1])
        ops = [TransformOp(b, c, h, w, src, dst, seed + i, rotate=True)
               for i, (c, h, w) in enumerate(TRANSFORM_SHAPES)]
        dom = max(range(len(ops)), key=lambda i: ops[i].bytes)
        desc = {"workload": f"BASELINE config 3: {LAYOUT_NAMES[src].upper()}->"
                            f"{LAYOUT_NAMES[dst].upper()} transform over the AlexNet + VGG-16 "
                            f"activation shapes, batch {b} per GPU",
                "batch_per_gpu": b, "global_batch": b * world, "parallelism": par,
                "shapes": [f"{b}x{c}x{h}x{w}" for c, h, w in TRANSFORM_SHAPES],
                "l2_policy": "each step streams every shape once; shapes smaller than 2x L2 "
                             "rotate over enough copies to stream > 4x L2 between reuses"}
        return Workload(ops, ops, desc, dom, "weak", b * world, "images")
    raise SystemExit(f"unknown workload {name}")


# ---------------------------------------------------------------- clocks ---
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


class ClockSampler:
    """NVML polling thread (clocks.sm + throttle reasons) for the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], 0, False
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        names = [v for k, v in REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------ reference ----
def ref_sample_batch(ops, threads, budget_bytes):
    """Images per op for the reference timing: the full per-op batch (the
    same workload as our arm) unless `budget_bytes` > 0 bounds the sample's
    algorithmic bytes (CPU unit tests)."""
    full = min(op.units for op in ops)
    if not budget_bytes:
        return full
    per_image = sum(op.bytes / max(1, op.units) for op in ops)
    b = max(threads, int(budget_bytes // max(1.0, per_image)))
    b = max(threads, (b // threads) * threads)
    return min(b, full)


def time_reference(ops, threads, batch, steps, warmup):
    """Run every op's reference call on a `batch`-image sample per step;
    returns (GB/s over the timed steps, seconds per step, sample bytes)."""
    sessions = [op.ref_session(min(batch, op.units), threads) for op in ops]
    sample_bytes = sum(b for _, b in sessions)
    for _ in range(warmup):
        for s, _ in sessions:
            s.run()
    total = 0.0
    for _ in range(steps):
        for s, _ in sessions:
            total += s.run()
    for s, _ in sessions:
        s.close()
    return sample_bytes * steps / total / GB, total / steps, sample_bytes


def cpu_desc():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def sample_text(batch, full, threads, sample_bytes):
    what = "the full workload" if batch >= full else f"{batch} of {full} images per layer"
    return (f"{what}, N-sharded over {threads} std::threads calling the unmodified reference "
            f"function on their shard ({sample_bytes / GB:.3f} GB algorithmic per step)")


def run_reference_arm(args, rank, world):
    """--impl reference: the unmodified reference CPU path (oracle/_ref) on this
    host's cores, on the WHOLE job of our arm's config (the global batch for
    strong scaling); rank 0 only under torchrun.  Never loads
    paper_1610_03618_b200's CUDA library (the ops are shape-only)."""
    if rank != 0:
        return
    from oracle.oracle import Ref

    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/liblcnn_ref.so not built (needs /root/reference at build)"}))
        return
    threads = host_threads()
    wl = build_workload(args.workload, world, 0, args.plan)
    ops = wl.global_ops
    batch = ref_sample_batch(ops, threads, args.ref_sample_gb * GB)
    gbs, sec, sample_bytes = time_reference(ops, threads, batch, args.steps, args.warmup)
    line = {"metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3),
            "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (mt19937 uniform[-1,1), per-thread shard)", "config": wl.desc,
            "impl": "reference",
            "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads,
                             "kind": "reference", "cpu": cpu_desc(), "build": Ref.variant(),
                             "sample": sample_text(batch, min(op.units for op in ops), threads,
                                                   sample_bytes)},
            "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------- main -----
def free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


# Collective backend: NCCL (one GPU per rank).  LCNN_BENCH_BACKEND=gloo is a
# test mode for a box with fewer GPUs than ranks (ranks then share cuda:0 and
# the collectives run on host copies); its numbers are not scaling numbers.
BACKEND = os.environ.get("LCNN_BENCH_BACKEND", "nccl")


def all_reduce_max(dist, t):
    if BACKEND == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t
    h = t.cpu()
    dist.all_reduce(h, op=dist.ReduceOp.MAX)
    t.copy_(h)
    return t


def all_gather_flat(dist, out, t):
    if BACKEND == "nccl":
        dist.all_gather_into_tensor(out, t)
        return out
    parts = [torch_empty_like_cpu(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t.cpu())
    out.copy_(__import__("torch").cat(parts).to(out.device))
    return out


def torch_empty_like_cpu(t):
    return __import__("torch").empty(t.numel(), dtype=t.dtype)


def relaunch_distributed(gpus):
    """`bench.py --gpus N` without a torchrun environment: re-exec through
    torch.distributed.run with N local ranks (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench.py: launching {gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="vgg_pools",
                    help="vgg_pools (default, config 4) | vgg_pools_nchw | pl5[_nchw][_avg] | "
                         "softmax[_ROWS] | softmax5[_ROWS] | softmax_64k | softmax[5]_10k | softmax_cCOLS | "
                         "transform[_nchw|_nhwc|_hwcn][_N] | alexnet | alexnet_mixed | vgg16")
    ap.add_argument("--plan", type=int, nargs=2, default=None,
                    help="coarsening fh fw for every pool layer (default: the per-layer plans "
                         "measured on B200)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--ref-sample-gb", type=float, default=0.0,
                    help="bound the reference timing's algorithmic GB per step (0 = the full "
                         "workload, the default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ceiling", action="store_true",
                    help="skip the same-size device-copy ceiling of single-op workloads")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch single-kernel workloads one by one instead of a CUDA graph")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        relaunch_distributed(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.impl == "reference" else 1)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)

    if args.impl == "reference":
        if args.workload in NETWORKS:
            run_reference_network(args, rank, world)
        else:
            run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    count = torch.cuda.device_count()
    if count == 0:
        raise SystemExit("bench.py: no CUDA device visible")
    # one GPU per rank: LOCAL_RANK indexes the visible devices (a launcher
    # that masks each rank to one device leaves index 0)
    dev_index = local if local < count else local % count
    if world > count and count > 1 and BACKEND == "nccl":
        raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, {count} visible")
    torch.cuda.set_device(dev_index)
    device = torch.device("cuda", dev_index)
    if world > 1:
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(BACKEND)
        dist.barrier()  # creates the communicator
        print(f"bench.py: rank {rank}/{world} {BACKEND.upper()} communicator up on "
              f"cuda:{dev_index} (nranks={dist.get_world_size()})", file=sys.stderr, flush=True)

    def barrier():
        if world > 1:
            dist.barrier()

    if args.workload in NETWORKS:
        run_network_workload(args, torch, dist, rank, world, local, device, barrier)
        if world > 1:
            dist.destroy_process_group()
        return

    wl = build_workload(args.workload, world, rank, args.plan)
    ops = [op.alloc(torch, device) for op in wl.ops]
    dom = wl.dom
    stream = torch.cuda.current_stream(device)
    sh = stream.cuda_stream
    step_bytes = sum(op.bytes for op in ops)

    def step():
        for op in ops:
            op.launch(sh)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()

    K = args.steps
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # The K steps are captured into one CUDA graph so host launch gaps do not
    # count (single-kernel workloads -- PL5 184 MB, softmax 32 MB -- and the
    # small-N transform sweep last microseconds per launch).  A single-kernel
    # workload's dominant kernel is its only kernel (avg = region / K); in a
    # multi-kernel step the dominant kernel's launches are bracketed by
    # external timing events recorded INSIDE the captured graph, so they are
    # timed on its stream within the timed region.  If the capture fails, the
    # steps are plain stream launches with the same events.
    use_graph = not args.no_graph
    graph = None
    dev_ev = [(torch.cuda.Event(enable_timing=True, external=use_graph),
               torch.cuda.Event(enable_timing=True, external=use_graph))
              for _ in range(0 if use_graph and len(ops) == 1 else K)]

    def timed_launches(s, sh_):
        for i in range(K):
            for j, op in enumerate(ops):
                if j == dom and dev_ev:
                    dev_ev[i][0].record(s)
                    op.launch(sh_)
                    dev_ev[i][1].record(s)
                else:
                    op.launch(sh_)

    if use_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(device)
            cap.wait_stream(stream)
            with torch.cuda.graph(graph, stream=cap):
                timed_launches(cap, cap.cuda_stream)
            stream.wait_stream(cap)
            graph.replay()  # warm the graph once
            torch.cuda.synchronize()
        except Exception as e:  # capture unsupported: plain stream launches
            print(f"bench.py: graph capture failed ({str(e)[:80]}), stream launches", file=sys.stderr)
            torch.cuda.synchronize()
            graph, use_graph = None, False
            dev_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(K)]
        barrier()

    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ selects these launches
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        if use_graph:
            graph.replay()
        else:
            timed_launches(stream, sh)
        ev1.record(stream)
        torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    barrier()
    ms = ev0.elapsed_time(ev1)
    dom_ms = ms / K if not dev_ev else sum(a.elapsed_time(b) for a, b in dev_ev) / K
    t = torch.tensor([ms, dom_ms], device=device, dtype=torch.float64)
    if world > 1:
        all_reduce_max(dist, t)
    ms, dom_ms = float(t[0]), float(t[1])
    # multi-kernel steps: the dominant kernel also timed alone (a graph of K
    # launches of it, no event nodes between them) -- for small kernels the
    # in-graph event nodes themselves cost microseconds
    iso_ms = None
    if use_graph and len(ops) > 1:
        g_dom = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device)
        cap.wait_stream(stream)
        with torch.cuda.graph(g_dom, stream=cap):
            for _ in range(K):
                ops[dom].launch(cap.cuda_stream)
        stream.wait_stream(cap)
        g_dom.replay()
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        g_dom.replay()
        d1.record(stream)
        torch.cuda.synchronize()
        iso_ms = d0.elapsed_time(d1) / K
    # whole-job bytes: the global batch for strong scaling, world x per-GPU for weak
    job_bytes = wl.step_bytes_global if wl.scaling == "strong" else step_bytes * world
    value = job_bytes * K / (ms / 1e3) / GB

    peak, peak_src = load_peaks()
    dom_op = ops[dom]
    achieved = dom_op.bytes / (dom_ms / 1e3) / GB
    traffic = load_traffic(args.workload)
    roofline = {"bound": "hbm", "kernel": dom_op.name, "achieved": round(achieved, 1),
                "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "algorithmic_bytes_per_launch": dom_op.bytes,
                "avg_launch_ms": round(dom_ms, 5),
                "traffic": traffic if world == 1 else None,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full, N=1 shapes)",
                "step_frac": round(step_bytes / (ms / K / 1e3) / GB / peak, 4)}
    if iso_ms:
        roofline["isolated"] = {"avg_launch_ms": round(iso_ms, 5),
                                "achieved": round(dom_op.bytes / (iso_ms / 1e3) / GB, 1),
                                "what": "the dominant kernel alone: one CUDA graph of K launches"}

    # ---- size ceiling: a plain device copy of the same bytes, same harness ----
    ceiling = None
    if use_graph and dom_op.in_bytes == dom_op.out_bytes and not args.no_ceiling:
        ceiling = copy_ceiling(torch, device, dom_op, K,
                               roofline["isolated"]["achieved"] if iso_ms else achieved)

    # ---- e2e: host buffers through the C ABI (pinned H2D, kernel, D2H) ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(torch, device, ops, world, args.e2e_steps, barrier, dist,
                      wl.step_bytes_global if wl.scaling == "strong" else None)

    # ---- cpu baseline: reference CPU path, rank 0 at N=1 only ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import Ref

            if Ref.available():
                threads = host_threads()
                b = ref_sample_batch(wl.global_ops, threads, args.ref_sample_gb * GB)
                gbs, sec, sb = time_reference(wl.global_ops, threads, b, 3, 1)
                cpu = {"value": round(gbs, 3), "unit": "GB/s", "cores": threads,
                       "kind": "reference", "cpu": cpu_desc(), "build": Ref.variant(),
                       "sample": sample_text(b, min(op.units for op in wl.global_ops), threads,
                                             sb) + "; mean of 3 steps after 1 warm-up"}
        except Exception as e:  # the baseline must never hide the GPU number
            cpu = {"value": None, "error": str(e)}

    clk = clocks.summary()
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
                "steps": K, "warmup": args.warmup, "ms_per_step": round(ms / K, 4),
                "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (uniform[-1,1) from torch's on-device RNG)",
                "config": wl.desc,
                "kernels": [op.name for op in ops],
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "copy_ceiling": ceiling,
                "gpu_launches": K * len(ops), "clocks": clk, "impl": "ours",
                "timing": ("one CUDA graph of K steps" + ("" if len(ops) == 1 else
                           "; dominant kernel: external CUDA events around its launches "
                           "inside the graph") if use_graph else "stream launches")}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def copy_ceiling(torch, device, op, K, achieved):
    """What a plain device copy of the op's bytes reaches in the same harness:
    one CUDA graph of K copies over the same rotated buffers, read in_bytes +
    write out_bytes per launch, by (a) cudaMemcpyAsync device-to-device
    (torch copy_ of contiguous fp32) and (b) torch's vectorised elementwise
    kernel (y = x * 1).  For a small single launch (the 4096 x 1000
    classifier moves 32.8 MB) the launch and ramp cost is part of every step,
    so the faster of the two -- not the streaming copy peak -- is the ceiling
    a kernel of that size reaches here."""
    stream = torch.cuda.current_stream(device)
    n = op.in_bytes // 4
    res = {}
    for tag, fn in (("memcpy_d2d", lambda src, dst: dst.copy_(src)),
                    ("elementwise", lambda src, dst: torch.mul(src, 1.0, out=dst))):
        def one(i):
            r = i % op.rot
            fn(op.x[r * n:(r + 1) * n], op.y[r * n:(r + 1) * n])

        for i in range(3):
            one(i)
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device)
        cap.wait_stream(stream)
        with torch.cuda.graph(graph, stream=cap):
            for i in range(K):
                one(i)
        stream.wait_stream(cap)
        graph.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        graph.replay()
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / K
        res[tag] = {"GBps": round(op.bytes / (ms / 1e3) / GB, 1), "avg_launch_ms": round(ms, 5)}
    best = max(v["GBps"] for v in res.values())
    return {"what": "same bytes, same rotated buffers, one CUDA graph of K launches "
                    "(size ceiling incl. per-launch cost)",
            "variants": res, "value": best, "unit": "GB/s",
            "kernel_frac_of_ceiling": round(achieved / best, 4)}


def run_e2e(torch, device, ops, world, steps, barrier, dist, job_bytes=None):
    """Same metric through the C ABI with HOST buffers: every step copies each
    layer's input from pinned host memory (H2D stream), runs the kernel
    (compute stream) and copies the result back (D2H stream); the two copy
    engines overlap across layers.  Timed with events on the issuing streams,
    max over ranks.  This is the best case for host buffers (pinned memory,
    copies overlapped with kernels); the lcnn:: value-semantics API
    (host/src/ops.cpp: pageable upload, kernel, download per call) is slower."""
    comp = torch.cuda.current_stream(device)
    h2d = torch.cuda.Stream(device)
    d2h = torch.cuda.Stream(device)
    hx = [op.next_views()[0].cpu().pin_memory() for op in ops]
    hy = [torch.empty(op.out_bytes // 4, dtype=torch.float32).pin_memory() for op in ops]
    h2d_bytes = sum(op.in_bytes for op in ops)
    d2h_bytes = sum(op.out_bytes for op in ops)

    # Per-layer ordering only (no drain between steps): step i+1's H2D into a
    # layer's input waits for step i's kernel of that layer, and a kernel waits
    # for step i's D2H of its output buffer -- so the H2D engine streams
    # continuously across steps.
    kdone = [None] * len(ops)  # kernel of layer j finished (its input may be overwritten)
    odone = [None] * len(ops)  # D2H of layer j finished (its output may be overwritten)

    def one_step():
        done_in = []
        views = [op.next_views() for op in ops]
        for j, ((dx, _), x) in enumerate(zip(views, hx)):
            if kdone[j] is not None:
                h2d.wait_event(kdone[j])
            with torch.cuda.stream(h2d):
                dx.copy_(x, non_blocking=True)
                e = torch.cuda.Event()
                e.record(h2d)
            done_in.append(e)
        for j, (op, (_, dy), e, y) in enumerate(zip(ops, views, done_in, hy)):
            comp.wait_event(e)
            if odone[j] is not None:
                comp.wait_event(odone[j])
            op.launch(comp.cuda_stream)
            k = torch.cuda.Event()
            k.record(comp)
            kdone[j] = k
            d2h.wait_event(k)
            with torch.cuda.stream(d2h):
                y.copy_(dy, non_blocking=True)
                o = torch.cuda.Event()
                o.record(d2h)
            odone[j] = o

    one_step()  # warm-up (page-locked paths, allocator)
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    h2d.wait_stream(comp)
    e0.record(comp)
    h2d.wait_stream(comp)
    for _ in range(steps):
        one_step()
    comp.wait_stream(d2h)  # the region ends when the last result is back on the host
    comp.wait_stream(h2d)
    e1.record(comp)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=device, dtype=torch.float64)
    if world > 1:
        all_reduce_max(dist, t)
    ms = float(t[0])
    step_bytes = job_bytes or sum(op.bytes for op in ops) * world
    value = step_bytes * steps / (ms / 1e3) / GB
    return {"value": round(value, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d_bytes,
            "d2h_bytes_per_step": d2h_bytes, "steps": steps, "ms_per_step": round(ms / steps, 3),
            "path": "pinned host -> cudaMemcpyAsync H2D -> lcnn_* C ABI kernel -> D2H, "
                    "copy engines overlapped across layers and steps (per-layer events, no "
                    "drain between steps; best-case pinned pipeline; h2d/d2h bytes are per GPU)"}


# ------------------------------------------------------ whole networks ---
NETWORKS = {
    "alexnet": (os.path.join(ROOT, "configs", "alexnet.json"),
                "BASELINE config 5: whole AlexNet forward (conv/pool/fc/softmax chain of SURVEY "
                "8d), 128 images per GPU"),
    "alexnet_mixed": (os.path.join(ROOT, "configs", "alexnet_mixed.json"),
                      "BASELINE config 5 with the paper's mixed per-layer assignment "
                      "(test_net.cpp:186-209: conv2, conv4, conv5 NCHW, the rest CHWN; 4 "
                      "inserted transforms), 128 images per GPU"),
    "vgg16": (os.path.join(ROOT, "configs", "vgg16.json"),
              "whole VGG-16 forward (13 conv 3x3, 5 max pools, 3 fc, softmax), 128 images per "
              "GPU (the AlexNet/VGG forward of the north star)"),
}


def layer_flops(cfg, weights=False):
    """name -> forward flops of one image for every conv / fc layer of a
    network config (shapes inferred as net.cpp infer_shapes does); with
    weights=True, the total weight count instead."""
    c, h, w = cfg["input"]["c"], cfg["input"]["h"], cfg["input"]["w"]
    flat = None
    out = {}
    nw = 0
    for L in cfg["layers"]:
        k = L["kind"]
        if k == "conv":
            f, s, p, co = L["f"], L.get("stride", 1), L.get("pad", 0), L["c_out"]
            ho, wo = (h + 2 * p - f) // s + 1, (w + 2 * p - f) // s + 1
            out[L["name"]] = 2.0 * co * ho * wo * c * f * f
            nw += co * c * f * f
            c, h, w = co, ho, wo
        elif k == "pool":
            win, s = L["win"], L.get("stride", L["win"])
            h, w = (h - win) // s + 1, (w - win) // s + 1
        elif k == "fc":
            kk = flat if flat is not None else c * h * w
            out[L["name"]] = 2.0 * kk * L["out"]
            nw += kk * L["out"]
            flat = L["out"]
    return nw if weights else out


def thresholds():
    """B200 (c_t, n_t) from the calibration record if one was made on this
    hardware (profiles/b200_calibration.txt), else the titan-black preset."""
    path = os.path.join(ROOT, "profiles", "b200_calibration.txt")
    try:
        with open(path) as f:
            parts = dict(kv.split("=", 1) for kv in f.readline().split())
        return (int(parts["c_t"]), int(parts["n_t"]),
                "calibrated on B200 (profiles/b200_calibration.txt)")
    except Exception:
        return 32, 128, "titan-black preset"


def network_desc(workload, world):
    """The config dict both arms print for a whole-network workload."""
    cfg_path, workload_desc = NETWORKS[workload]
    cfg = json.loads(open(cfg_path).read())
    batch = cfg["input"]["n"]
    c_t, n_t, th_src = thresholds()
    weight_mb = layer_flops(cfg, weights=True) * 4 / 1e6
    return {"workload": workload_desc, "batch_per_gpu": batch, "global_batch": batch * world,
            "parallelism": f"N-shard x{world}, NCCL all_gather of logits only",
            "thresholds": [c_t, n_t], "thresholds_source": th_src,
            "l2_policy": f"activations + {weight_mb:.0f} MB of weights per step (> L2)"}


def run_network_workload(args, torch, dist, rank, world, local, device, barrier):
    """Whole-network forward (BASELINE config 5 AlexNet, 128 images per GPU =
    batch 1024 at 8 GPUs; or VGG-16), per-layer layout selection, conv/fc on
    tcgen05 (TF32)."""
    from paper_1610_03618_b200 import capi, netapi

    cfg_path, workload_desc = NETWORKS[args.workload]
    text = open(cfg_path).read()
    flops = layer_flops(json.loads(text))
    weight_mb = layer_flops(json.loads(text), weights=True) * 4 / 1e6
    batch = json.loads(text)["input"]["n"]
    c_t, n_t, th_src = thresholds()
    net = netapi.Network(text, c_t, n_t, seed=42, precision=capi.PREC_TF32)
    info = net.info(1)
    in_layout = info["first_layout"]
    rows, cols = info["out"]
    g = torch.Generator(device=device).manual_seed(7 + rank)
    dn, dc, dh, dw = info["dims"]
    x = torch.rand(dn * dc * dh * dw, device=device, generator=g) * 2 - 1
    y = torch.empty(rows * cols, device=device)
    stream = torch.cuda.current_stream(device)
    sh = stream.cuda_stream
    for _ in range(args.warmup):
        net.forward(x.data_ptr(), in_layout, y.data_ptr(), sh)
    torch.cuda.synchronize()
    # The forward replayed from the network's own CUDA graph
    # (lcnn_net_forward_graph: captured once for these buffers; stream-ordered
    # allocations become graph memory nodes, PDL edges stay programmatic): the
    # host issues one call per step instead of ~11-30 launches plus tensor-map
    # encodes, so a slow host CPU cannot open gaps between layers.  Checked
    # against a stream forward first.
    use_graph, graph_note = False, "stream launches (--no-graph)"
    if not args.no_graph:
        ref = y.clone()
        try:
            y.zero_()
            net.forward_graph(x.data_ptr(), in_layout, y.data_ptr(), sh)
            torch.cuda.synchronize()
            if torch.allclose(y, ref, rtol=1e-4, atol=1e-6):
                use_graph = True
                graph_note = ("lcnn_net_forward_graph: the network's cached CUDA graph of one "
                              "forward, replayed K times")
            else:
                graph_note = "stream launches (graph replay disagreed with the stream forward)"
        except Exception as e:  # capture unsupported: keep stream launches
            graph_note = f"stream launches (graph capture failed: {str(e)[:80]})"
            torch.cuda.synchronize()
        for _ in range(2):
            (net.forward_graph if use_graph else net.forward)(x.data_ptr(), in_layout,
                                                              y.data_ptr(), sh)
        torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    K = args.steps
    torch.cuda.nvtx.range_push("timed")
    with ClockSampler(local) as clocks:
        e0.record(stream)
        fwd = net.forward_graph if use_graph else net.forward
        for _ in range(K):
            fwd(x.data_ptr(), in_layout, y.data_ptr(), sh)
        e1.record(stream)
        torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    barrier()
    t = torch.tensor([e0.elapsed_time(e1)], device=device, dtype=torch.float64)
    if world > 1:
        all_reduce_max(dist, t)
    ms = float(t[0])
    value = batch * world * K / (ms / 1e3)

    # kernels one forward launches (CUPTI, outside the timed region)
    per_fwd = count_kernels(torch, lambda: net.forward(x.data_ptr(), in_layout, y.data_ptr(), sh))

    # per-entry device times of one forward (dominant kernel = slowest entry):
    # a ~10 ms sleep kernel ahead of each profiled forward lets the host queue
    # every launch before the GPU reaches them, so an entry's event span is
    # device time only (no host gaps); median of 5 forwards per entry
    runs = []
    for _ in range(5):
        torch.cuda._sleep(20_000_000)
        runs.append(net.profile(x.data_ptr(), in_layout, sh))
    prof = [(runs[0][i][0], statistics.median(r[i][1] for r in runs)) for i in range(len(runs[0]))]
    name, ns = max(prof, key=lambda e: e[1])
    fl = flops.get(name, 0.0) * batch
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    tf32_peak = float(peaks["bf16_tflops"]) / 2
    achieved = fl / (ns * 1e-9) / 1e12 if fl else None
    # the tensor pipe's own TF32 rate, measured with back-to-back M=128 N=256
    # tcgen05.mma on resident operands (scripts/mma_bench.cu, no memory traffic)
    mma_peak = None
    try:
        import re as _re

        rates = [float(m.group(1)) for m in _re.finditer(
            r"N=256\s+\S+ cyc/MMA\s+(\S+) TF/s",
            open(os.path.join(ROOT, "profiles", "r01_mma_bench.txt")).read())]
        mma_peak = max(rates) if rates else None
    except Exception:
        pass
    # peak: the measured TF32 tensor-pipe rate (cuBLAS bf16 / 2 understates
    # it on this part: our kind::tf32 N=256 MMAs issue at 1111 TF/s, above
    # half the library's bf16 burst); the bf16/2 figure is kept beside it
    peak = mma_peak or tf32_peak
    # a conv whose max pool runs in its epilogue (Network fuse_pools): the
    # pool's own entry is an empty span right after it
    ix = [e[0] for e in prof].index(name)
    fused = (ix + 1 < len(prof) and prof[ix + 1][0].startswith("pool") and
             prof[ix + 1][1] < 0.02 * ns)
    label = (f"{name} + {prof[ix + 1][0]} (tcgen05 kind::tf32 implicit GEMM, max pool fused "
             "into the epilogue)") if fused else f"{name} (tcgen05 kind::tf32 implicit GEMM)"
    roofline = {"bound": "tensor", "kernel": label,
                "achieved": round(achieved, 1) if achieved else None, "peak": peak,
                "peak_source": ("measured tcgen05.mma kind::tf32 M=128 N=256 issue rate, 148 SMs "
                                "(scripts/mma_bench.cu, profiles/r01_mma_bench.txt)") if mma_peak
                else "measured bf16 burst (MEASURED_PEAKS.json) / 2 = dense TF32",
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4) if achieved else None,
                "traffic": (load_traffic(args.workload) or {}).get(name),
                "peak_bf16_half": tf32_peak,
                "frac_of_bf16_half": round(achieved / tf32_peak, 4) if achieved else None,
                "avg_launch_ms": round(ns / 1e6, 4),
                "forward_tflops": round(info["flops_per_image"] * batch / (ms / K / 1e3) / 1e12, 1),
                "per_entry_us": {k: round(v / 1e3, 1) for k, v in prof}}

    # verification collective: gather every rank's logits (row-major concat)
    torch.cuda.synchronize()
    ok_rows = bool(torch.allclose(y.view(rows, cols).double().sum(1),
                                  torch.ones(rows, device=device, dtype=torch.float64), atol=1e-4))
    if world > 1:
        gathered = torch.empty(world * rows * cols, device=device)
        all_gather_flat(dist, gathered, y)
        ok_rows = ok_rows and bool(torch.equal(gathered.view(world, -1)[rank], y))
    # end to end: host buffers through lcnn_net_forward_host_many -- every
    # batch's H2D (pinned) and logits D2H inside the timed region; batch i+1's
    # H2D overlaps batch i's forward (two device input slots)
    e2e = None
    if not args.no_e2e:
        hx = [x.cpu().pin_memory(), (x.flip(0)).cpu().pin_memory()]
        hy = [torch.empty(rows * cols).pin_memory() for _ in range(2)]
        steps = max(4, min(args.e2e_steps * 4, K))
        ins = [hx[i % 2].data_ptr() for i in range(steps)]
        outs = [hy[i % 2].data_ptr() for i in range(steps)]
        net.forward_host_many(ins[:2], in_layout, outs[:2])  # warm-up
        barrier()
        t0 = time.perf_counter()
        net.forward_host_many(ins, in_layout, outs)
        dt = torch.tensor([time.perf_counter() - t0], device=device, dtype=torch.float64)
        if world > 1:
            all_reduce_max(dist, dt)
        # hy[0] holds the last even batch, whose input hx[0] is x (stream-K
        # tiles add in any order, so compare within the tf32 logits tolerance)
        ok_e2e = bool(torch.allclose(hy[0], y.cpu(), rtol=1e-3, atol=1e-6))
        e2e = {"value": round(batch * world * steps / float(dt[0]), 1), "unit": "images/s",
               "h2d_bytes_per_step": hx[0].numel() * 4, "d2h_bytes_per_step": hy[0].numel() * 4,
               "steps": steps, "ms_per_step": round(1e3 * float(dt[0]) / steps, 3),
               "logits_match_device_path": ok_e2e,
               "path": "lcnn_net_forward_host_many (pinned host -> H2D on a copy stream, "
                       "overlapped with the previous batch's forward -> D2H of the logits)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = reference_network_sample(cfg_path, c_t, n_t)
        except Exception as e:
            cpu = {"value": None, "error": str(e)}
    if rank == 0:
        layouts = [capi.LAYOUT_NAMES.get(l, "-") for l in net.layouts[:12]]
        line = {"metric": METRIC, "value": round(value, 1), "unit": "images/s", "n_gpus": world,
                "steps": K, "warmup": args.warmup, "ms_per_step": round(ms / K, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "tf32",
                "data": "synthetic (uniform[-1,1) input, reference-seeded weights)",
                "config": network_desc(args.workload, world),
                "network": {"layouts": layouts, "transforms": info["transforms"],
                            "logits_rows_sum_to_1": ok_rows},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": per_fwd * K if per_fwd is not None else None,
                "gpu_launches_per_step": per_fwd, "clocks": clocks.summary(), "impl": "ours",
                "timing": graph_note}
        print(json.dumps(line))


def count_kernels(torch, fn):
    """Kernel launches of fn() as recorded by CUPTI (torch.profiler); memsets
    and copies are not kernels.  None if the profiler is unavailable."""
    try:
        from torch.profiler import ProfilerActivity, profile

        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as p:
            fn()
            torch.cuda.synchronize()
        names = [e.name for e in p.events() if e.device_type.name == "CUDA"]
        return sum(1 for n in names if "memset" not in n.lower() and "memcpy" not in n.lower())
    except Exception:
        return None


def reference_network_sample(cfg_path, c_t, n_t, batch_per_thread=1):
    from oracle.oracle import Ref, ref_time_network

    if not Ref.available():
        return None
    threads = host_threads()
    cfg = json.loads(open(cfg_path).read())
    cfg["input"]["n"] = batch_per_thread
    sec = ref_time_network(json.dumps(cfg), c_t, n_t, threads)
    return {"value": round(batch_per_thread * threads / sec, 3), "unit": "images/s",
            "cores": threads, "kind": "reference", "cpu": cpu_desc(),
            "sample": f"{batch_per_thread} image(s) per std::thread x {threads} threads through "
                      f"the unmodified run_network ({sec:.2f} s)"}


def run_reference_network(args, rank, world):
    if rank != 0:
        return
    from oracle.oracle import Ref

    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    c_t, n_t, _ = thresholds()
    total_img, total_s, timed = 0, 0.0, 0
    cfg_path, workload_desc = NETWORKS[args.workload]
    t_start = time.perf_counter()
    # a step is one image per host thread through the unmodified run_network;
    # at most 2 warm-up steps, and the timed steps stop after ~150 s of CPU
    # work (a VGG-16 step takes ~25 s on 16 threads)
    for i in range(min(args.warmup, 2) + args.steps):
        r = reference_network_sample(cfg_path, c_t, n_t)
        if i >= min(args.warmup, 2):
            total_img += r["cores"]
            total_s += r["cores"] / r["value"]
            timed += 1
            if time.perf_counter() - t_start > 150:
                break
    v = total_img / total_s
    threads = host_threads()
    print(json.dumps({"metric": METRIC, "value": round(v, 3), "unit": "images/s",
                      "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": round(1e3 * total_s / args.steps, 1),
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                      "dtype": "f32", "data": "synthetic", "impl": "reference",
                      "config": network_desc(args.workload, world),
                      "cpu_baseline": {"value": round(v, 3), "unit": "images/s", "cores": threads,
                                       "kind": "reference", "cpu": cpu_desc(),
                                       "build": Ref.variant(),
                                       "sample": f"1 image per thread x {threads} threads, "
                                                 f"{timed} timed step(s)"},
                      "e2e": {"value": round(v, 3), "unit": "images/s", "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0}}))


if __name__ == "__main__":
    main()
