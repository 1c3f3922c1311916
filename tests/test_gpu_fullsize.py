"""Full-size parity of every configuration bench.py measures,
with the kernels and plans exactly as benched.

* Single-op workloads (configs 1-4): bench.build_workload's own ops are
  allocated and launched once, and every output is compared with the
  reference-pinned C oracle on the same input -- bit-exact for pooling and
  transforms, approx_equal 1e-6 (the reference's bar) for softmax.
* Whole networks (config 5 AlexNet, VGG-16): the benched batch of 128 runs
  through lcnn_net_forward in the benched precision; a 16-image slice of the
  logits is compared with the UNMODIFIED reference run_network on those
  images, N-sharded over host threads (batch independence,
  test_conv.cpp:117-141).  Tolerances on the softmax output p:
    FP32 : approx_equal 1e-5 (test_net.cpp:211-248) and |log p - log p_ref|
           <= 1e-4;
    TF32 : |log p - log p_ref| <= 5e-3, i.e. 0.5 % relative on every
           probability.  For scale: the reference's own log-probabilities
           spread over ~0.1 across the 1000 classes with these seeded weights,
           and tf32 truncates each operand by < 2^-10 relative.
* Full-size convolution routes: AlexNet conv1 (SHARE, 128x3x227^2 f11/s4),
  VGG conv1_1 and conv1_2 (128 images at 224^2) run on the whole batch; a
  slice of images is compared with a float64 reference under the TF32 bound
  2^-9 * (|x| conv |w|) + 1e-6, and one image with the C oracle."""
import json
import os

import numpy as np
import pytest

import bench
from oracle.oracle import CHWN, NCHW, C, Ref, approx_equal, bit_equal, rng_uniform
from paper_1610_03618_b200 import capi, lcnn, netapi

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run_ops(cuda, name):
    import torch

    wl = bench.build_workload(name, 1, 0)
    ops = [op.alloc(torch, cuda) for op in wl.ops]
    sh = torch.cuda.current_stream(cuda).cuda_stream
    for op in ops:
        op.launch(sh)
    torch.cuda.synchronize()
    return ops


def _release(torch):
    import gc

    gc.collect()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["vgg_pools", "vgg_pools_nchw", "pl5", "pl5_nchw"])
def test_bench_pool_workloads_bit_exact(cuda, name):
    import torch

    ops = _run_ops(cuda, name)
    for op in ops:
        assert op._i == 1
        x = op.x[:op.in_bytes // 4].cpu().numpy()
        y = op.y[:op.out_bytes // 4].cpu().numpy()
        want, _ = C.pool_plain(x, op.n, op.c, op.h, op.w, op.layout, op.win, op.win, op.stride,
                               op.avg)
        assert bit_equal(y, want), op.name
        del x, y, want
    del ops
    _release(torch)


@pytest.mark.parametrize("name", ["softmax", "softmax5", "softmax_64k", "softmax_128"])
def test_bench_softmax_workloads(cuda, name):
    import torch

    (op,) = _run_ops(cuda, name)
    x = op.x[:op.rows * op.cols].cpu().numpy()
    y = op.y[:op.rows * op.cols].cpu().numpy()
    want = (C.softmax_fused(x, op.rows, op.cols)[0] if op.fused
            else C.softmax_reference(x, op.rows, op.cols)[0])
    assert approx_equal(y, want, 1e-6), op.name
    assert int(op.flag.item()) == 0
    del op
    _release(torch)


@pytest.mark.parametrize("name", ["transform", "transform_nchw_256", "transform_32",
                                  "transform_nchw_64"])
def test_bench_transform_workloads_bit_exact(cuda, name):
    import torch

    ops = _run_ops(cuda, name)
    for op in ops:
        x = op.x[:op.in_bytes // 4].cpu().numpy()
        y = op.y[:op.out_bytes // 4].cpu().numpy()
        assert bit_equal(y, C.transform(x, op.n, op.c, op.h, op.w, op.src, op.dst)), op.name
    del ops
    _release(torch)


def _slice_vs_reference(cuda, cfg_name, precision, slice_n=16):
    """Full benched batch on the GPU, first `slice_n` images vs the reference."""
    import torch

    text = open(os.path.join(ROOT, "configs", cfg_name)).read()
    cfg = json.loads(text)
    n = cfg["input"]["n"]
    c_t, n_t, _ = bench.thresholds()
    net = netapi.Network(text, c_t, n_t, seed=42, precision=precision)
    info = net.info(NCHW)
    rows, cols = info["out"]
    assert rows == n
    _, c, h, w = info["dims"]
    x = rng_uniform(2024, n * c * h * w)
    dx = torch.from_numpy(x).to(cuda)
    dy = torch.empty(rows * cols, device=cuda)
    net.forward(dx.data_ptr(), NCHW, dy.data_ptr(), torch.cuda.current_stream(cuda).cuda_stream)
    torch.cuda.synchronize()
    got = dy.cpu().numpy().reshape(rows, cols)[:slice_n]
    want = Ref.run_network_sharded(text, x[:slice_n * c * h * w], slice_n, c_t, n_t, seed=42)
    net.close()
    assert np.allclose(got.sum(1), 1.0, atol=1e-5)
    return got, want


@pytest.mark.parametrize("precision", ["tf32", "fp32"])
def test_alexnet_forward_fullsize_vs_reference(cuda, precision):
    prec = capi.PREC_TF32 if precision == "tf32" else capi.PREC_FP32
    got, want = _slice_vs_reference(cuda, "alexnet.json", prec)
    dlog = np.abs(np.log(got.astype(np.float64)) - np.log(want.astype(np.float64))).max()
    if precision == "fp32":
        assert approx_equal(got, want, 1e-5) and dlog <= 1e-4, dlog
    else:
        assert dlog <= 5e-3, dlog


def test_alexnet_mixed_layouts_fullsize_vs_reference(cuda):
    """The paper's mixed per-layer assignment (test_net.cpp:186-209 mapped onto
    AlexNet: conv2/conv4/conv5 NCHW, 4 inserted transforms) at the benched
    size, against the reference running the same explicit layouts."""
    got, want = _slice_vs_reference(cuda, "alexnet_mixed.json", capi.PREC_TF32)
    dlog = np.abs(np.log(got.astype(np.float64)) - np.log(want.astype(np.float64))).max()
    assert dlog <= 5e-3, dlog
    text = open(os.path.join(ROOT, "configs", "alexnet_mixed.json")).read()
    net = netapi.Network(text, *bench.thresholds()[:2], seed=42, precision=capi.PREC_TF32)
    assert net.info(CHWN)["transforms"] == 4
    ref_layouts, steps = Ref.plan_network(text)
    assert [p for p, _, _ in steps] == [2, 3, 5, 7]
    assert net.layouts[:8] == ref_layouts[:8]
    net.close()


def test_vgg16_forward_fullsize_vs_reference(cuda):
    got, want = _slice_vs_reference(cuda, "vgg16.json", capi.PREC_TF32)
    dlog = np.abs(np.log(got.astype(np.float64)) - np.log(want.astype(np.float64))).max()
    assert dlog <= 5e-3, dlog


@pytest.mark.parametrize("geom", [
    # name, n, ci, h, co, f, stride, pad
    ("alexnet_conv1_share", 128, 3, 227, 96, 11, 4, 0),
    ("vgg_conv1_1", 128, 3, 224, 64, 3, 1, 1),
    ("vgg_conv1_2", 128, 64, 224, 64, 3, 1, 1),
    ("vgg_conv2_1", 128, 64, 112, 128, 3, 1, 1),
    ("vgg_conv2_2", 128, 128, 112, 128, 3, 1, 1),
])
def test_conv_routes_fullsize(cuda, geom):
    import torch

    name, n, ci, h, co, f, st, pd = geom
    g = torch.Generator(device=cuda).manual_seed(5)
    x = torch.rand(n, ci, h, h, device=cuda, generator=g) * 2 - 1
    wt = (torch.rand(co, ci, f, f, device=cuda, generator=g) * 2 - 1).contiguous()
    t = lcnn.DeviceTensor4D(n, ci, h, h, CHWN, x.permute(1, 2, 3, 0).contiguous().reshape(-1))
    y = lcnn.conv_forward(t, wt, co, f, f, st, pd, lcnn.TF32)
    ho, wo = lcnn.conv_output_extents(h, h, f, f, st, pd)
    got = y.data.view(co, ho, wo, n)
    k = 8  # images checked against float64 (spread over the batch: 32-image groups)
    idx = torch.tensor([0, 1, 31, 32, 63, 64, 100, 127], device=cuda)[:k]
    xs = x.index_select(0, idx).double()
    want = torch.nn.functional.conv2d(xs, wt.double(), stride=st, padding=pd)
    bound = torch.nn.functional.conv2d(xs.abs(), wt.abs().double(), stride=st, padding=pd)
    gs = got.index_select(3, idx).permute(3, 0, 1, 2).double()
    err = (gs - want).abs()
    assert bool((err <= bound * 2.0 ** -9 + 1e-6).all()), (name, float(err.max()))
    # one image against the reference-pinned C oracle (NCHW in, NCHW out)
    x0 = x[127].contiguous().cpu().numpy().reshape(-1)
    w0 = wt.cpu().numpy().reshape(-1)
    ref = C.conv_oracle(x0, w0, 1, ci, h, h, NCHW, co, f, f, st, pd).astype(np.float64)
    refb = C.conv_oracle(np.abs(x0), np.abs(w0), 1, ci, h, h, NCHW, co, f, f, st, pd)
    g0 = got[..., 127].cpu().numpy().astype(np.float64).reshape(-1)
    assert np.all(np.abs(g0 - ref) <= refb * 2.0 ** -9 + 1e-6), name
    del x, y, got
    _release(torch)
