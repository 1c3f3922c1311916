"""GPU parity for the dense whole-network path: the tcgen05 implicit-GEMM
convolution (CHWN), the tcgen05 GEMM (fc layers), and the fp32 CUDA-core
kernels, against float64 references.

Stated tolerances, with B = (|x| conv |w|) or |A||B|
the magnitude bound of each output:
  FP32   : approx_equal 1e-5 against the fp64 oracle -- the reference's own
           bar (acceptance.cpp:113-118) -- or 2^-21 * B for very long K
           (fp32 16-deep partials + fp64 total, like gemm_blocked);
  3xTF32 : |y - y64| <= 2^-16 * B -- hi*hi + hi*lo + lo*hi removes the tf32
           operand rounding; what remains is the tensor core's truncating fp32
           accumulation, which grows linearly with K (measured on B200);
  TF32   : |y - y64| <= 2^-9 * B + 1e-6 -- two tf32 operand truncations
           (< 1 ulp = 2^-10 each) per product.
"""
import numpy as np
import pytest

from oracle.oracle import CHWN, NCHW, C, approx_equal, rng_uniform
from paper_1610_03618_b200 import lcnn

pytestmark = pytest.mark.gpu


def _torch_conv64(x_nchw, f, stride, pad):
    import torch

    return torch.nn.functional.conv2d(x_nchw.double(), f.double(), stride=stride, padding=pad)


def _check_conv(cuda, n, ci, h, w, co, f, stride, pad, layout, precision, seed=0):
    fh = fw = f
    import torch

    g = torch.Generator(device=cuda).manual_seed(seed)
    x = torch.rand(n, ci, h, w, device=cuda, generator=g) * 2 - 1
    f = torch.rand(co, ci, fh, fw, device=cuda, generator=g) * 2 - 1
    want = _torch_conv64(x, f, stride, pad)
    bound = _torch_conv64(x.abs(), f.abs(), stride, pad)
    xin = x if layout == NCHW else x.permute(1, 2, 3, 0).contiguous()
    t = lcnn.DeviceTensor4D(n, ci, h, w, layout, xin.reshape(-1))
    one_shot = lcnn.conv_forward(t, f.contiguous(), co, fh, fw, stride, pad, precision)
    # the pre-packed route (lcnn_conv_pack_filters + lcnn_conv_forward_packed)
    packed = lcnn.pack_conv_filters(t, f.contiguous(), co, fh, fw, stride, pad, precision)
    via_pack = lcnn.conv_forward_packed(t, packed, co, fh, fw, stride, pad, precision)
    ho, wo = want.shape[2], want.shape[3]
    for tag, out in (("one-shot", one_shot), ("packed", via_pack)):
        got = out.data.view(n, co, ho, wo) if layout == NCHW else \
            out.data.view(co, ho, wo, n).permute(3, 0, 1, 2)
        got = got.double()
        err = (got - want).abs()
        ok = bool((err <= tolerance(precision, got, want, bound)).all())
        assert ok, (tag, n, ci, h, w, co, fh, fw, stride, pad, layout, precision,
                    float(err.max()))
    if precision == lcnn.FP32:  # deterministic kernels: the two routes agree bit for bit
        assert torch.equal(one_shot.data, via_pack.data)


def tolerance(precision, got, want, bound):
    import torch

    if precision == lcnn.TF32:
        return bound * 2.0 ** -9 + 1e-6
    if precision == lcnn.X3TF32:
        return bound * 2.0 ** -16 + 1e-6
    scale = torch.maximum(torch.maximum(got.abs(), want.abs()), torch.ones_like(got))
    return torch.maximum(1e-5 * scale, bound * 2.0 ** -21)


CASES = [  # (n, ci, h, w, co, f, stride, pad)
    (32, 32, 9, 9, 64, 3, 1, 1),      # CI-mode K order
    (32, 64, 13, 13, 96, 3, 1, 1),
    (64, 3, 35, 35, 96, 11, 4, 0),    # conv1-like: ROW mode, 33 -> 40 k-rows per filter row
    (32, 96, 13, 13, 64, 5, 1, 2),    # WIN FP=8 (ci % 32 == 0 -> CI mode actually)
    (32, 16, 10, 10, 48, 5, 2, 2),    # WIN FP=8 (80 k-rows: too many for ROW)
    (32, 3, 12, 12, 20, 3, 1, 1),     # ROW row pairs, co < 32
    (128, 3, 33, 33, 64, 3, 1, 1),    # ROW row pairs, grouped boxes, odd H_o
    (64, 5, 20, 20, 48, 3, 1, 0),     # ROW row pairs, ungrouped, no padding
    (64, 3, 40, 40, 64, 3, 1, 1),     # ROW row pairs, quad-chunk stores + stream-K tail (chunk path)
    (128, 3, 24, 24, 64, 3, 1, 1),    # ROW row pairs, quad-chunk stores, whole tiles
    (128, 32, 6, 6, 160, 1, 1, 0),    # 1x1, co > 128
    (96, 64, 7, 7, 64, 3, 2, 0),
    (128, 384, 13, 13, 256, 3, 1, 1),  # conv4: 170 tiles -> 148 whole + stream-K tail
    (32, 5, 15, 15, 130, 7, 2, 3),     # ROW mode, 35 -> 40 k-rows, ragged channel tile
    # N % 128 == 0: grouped 5D input boxes (one box per 128-column block)
    (128, 3, 35, 35, 96, 11, 4, 0),    # conv1-like ROW, row width 11 -> 16 (48 k-rows), channels on M
    (256, 3, 19, 19, 64, 5, 2, 1),     # ROW, width 5 -> 8 (24 k-rows)
    (128, 5, 15, 15, 130, 7, 2, 3),    # ROW, width 7 -> 8 (40 k-rows), ragged channel tile
    (128, 16, 10, 10, 48, 5, 2, 2),    # WIN
    (256, 64, 7, 7, 64, 3, 2, 0),      # CI, two blocks per pixel
    # >= 4 waves of 256-column tiles: the CTA-pair (cta_group::2) kernel
    (128, 32, 27, 27, 192, 3, 1, 1),   # CI, conv2-like channel tile (N = 192, 96 per CTA)
    (128, 16, 27, 27, 48, 5, 1, 2),    # WIN
    # channel planes >= 4 MB: TAPS mode (one box per filter row serves all its taps)
    (128, 32, 92, 92, 64, 3, 1, 1),    # C_o 64: TAPS row pairs (rows oh, oh+1 on the two M halves)
    (128, 32, 91, 91, 48, 3, 1, 1),    # row pairs, odd H_o (last pair has one row), C_o 48
    (128, 64, 92, 92, 64, 5, 1, 2),    # row pairs, 5x5 (6 input rows per pair)
    (64, 32, 130, 130, 64, 3, 1, 0),   # row pairs, no padding
    (64, 32, 130, 130, 160, 3, 2, 1),  # stride 2, two channel tiles, 32-image groups x 2
    (32, 32, 182, 182, 128, 3, 1, 1),  # TAPS, two accumulators (rows oh, oh+1 share input boxes)
    (64, 64, 129, 131, 160, 3, 1, 1),  # two accumulators: odd H_o, ragged pixel block, 2 channel tiles
    (32, 32, 200, 190, 96, 5, 1, 2),   # two accumulators, 5x5 (6 input rows per pair)
    # CI, output rows >= 28, planes < 4 MB: TAPS-N (4-pixel x 32-image tiles on a CTA pair)
    (64, 32, 30, 30, 96, 3, 1, 1),     # C_o 96: 48-row filter halves per CTA
    (128, 64, 28, 28, 384, 3, 1, 1),   # two 192-channel tiles, two 64-image blocks
    (64, 32, 57, 57, 64, 3, 2, 1),     # stride 2, Wo 29: ragged last pixel block
    (64, 32, 32, 32, 128, 5, 1, 2),    # 5x5: one box serves 5 taps
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("precision", [0, 1, 2])
def test_conv_chwn(cuda, case, precision):
    _check_conv(cuda, *case, CHWN, precision)


def test_conv_tapsn_forced_on_alexnet_shapes(cuda):
    """TAPS-N forced (LCNN_CONV_TAPSN=1, read once per process: a subprocess)
    on the AlexNet conv2-5 shapes the router keeps on the CI kernels."""
    import os
    import subprocess
    import sys

    code = (
        "import sys, torch; sys.path.insert(0, 'tests'); sys.path.insert(0, '.');"
        "import test_gpu_conv_gemm as t; from paper_1610_03618_b200 import lcnn;"
        "d = torch.device('cuda:0');"
        "[t._check_conv(d, *c, t.CHWN, lcnn.TF32) for c in ["
        "(128, 96, 27, 27, 192, 5, 1, 2), (128, 192, 13, 13, 384, 3, 1, 1),"
        "(128, 384, 13, 13, 256, 3, 1, 1), (64, 32, 13, 13, 96, 3, 1, 1)]];"
        "print('ok')")
    env = dict(os.environ, LCNN_CONV_TAPSN="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("case", CASES[:11] + [(128, 96, 27, 27, 192, 5, 1, 2)])
@pytest.mark.parametrize("precision", [0, 1])
def test_conv_nchw_via_chwn(cuda, case, precision):
    """NCHW on the tensor cores: NCHW->CHWN transpose, the CHWN route of the
    geometry, CHWN->NCHW transpose of the output (one-shot and packed)."""
    _check_conv(cuda, *case, NCHW, precision)


def test_conv_nchw_gather_kernel_still_correct(cuda):
    """The NCHW gather-producer kernel (LCNN_CONV_NCHW=gather, read once per
    process: a subprocess) stays parity-green as the measured alternative."""
    import os
    import subprocess
    import sys

    code = (
        "import sys, torch; sys.path.insert(0, 'tests'); sys.path.insert(0, '.');"
        "import test_gpu_conv_gemm as t; from paper_1610_03618_b200 import lcnn;"
        "d = torch.device('cuda:0');"
        "[t._check_conv(d, *c, t.NCHW, lcnn.TF32) for c in ["
        "(32, 96, 27, 27, 64, 5, 1, 2), (16, 3, 35, 35, 32, 11, 4, 0), (5, 3, 9, 9, 7, 3, 1, 1)]];"
        "print('ok')")
    env = dict(os.environ, LCNN_CONV_NCHW="gather")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("case", [(5, 3, 9, 9, 7, 3, 1, 1), (3, 4, 11, 11, 6, 5, 2, 2),
                                  (32, 8, 13, 13, 16, 3, 1, 1), (7, 2, 7, 7, 5, 1, 1, 0)])
@pytest.mark.parametrize("precision", [0, 2])
def test_conv_nchw_and_odd_batches(cuda, case, precision):
    _check_conv(cuda, *case, NCHW, precision)
    _check_conv(cuda, *case, CHWN, precision)


def test_conv_reference_fixtures(cuda, ref_vectors):
    """conv_oracle outputs from the reference binary (tests/golden)."""
    import torch

    v = ref_vectors
    keys = sorted({k.split("_")[1] for k in v.files if k.startswith("conv_")}, key=int)
    for k in keys:
        n, ci, h, w, co, f, stride, pad = v[f"conv_{k}_meta"].tolist()
        x = v[f"conv_{k}_in"]
        filt = torch.from_numpy(v[f"conv_{k}_filt"]).to(cuda)
        for layout in (NCHW, CHWN):
            xin = x if layout == NCHW else C.transform(x, n, ci, h, w, NCHW, CHWN)
            t = lcnn.DeviceTensor4D.from_host(xin, n, ci, h, w, layout, device=cuda)
            for prec in (lcnn.FP32,):
                out = lcnn.conv_forward(t, filt, co, f, f, stride, pad, prec)
                got = out.to_host()
                if layout == CHWN:
                    ho = (h + 2 * pad - f) // stride + 1
                    wo = (w + 2 * pad - f) // stride + 1
                    got = C.transform(got, n, co, ho, wo, CHWN, NCHW)
                assert approx_equal(got, v[f"conv_{k}_oracle"], 1e-5), (k, layout, prec)


@pytest.mark.parametrize("m,n,k", [(128, 128, 128), (96, 300, 64), (257, 129, 200),
                                   (128, 4096, 9216), (1000, 128, 4096), (33, 17, 13),
                                   (64, 1000, 4096),
                                   (1280, 4352, 640),   # 170 tiles: data-parallel wave + stream-K
                                   (2432, 1024, 96),    # 76 tiles, 3 k-blocks: pure stream-K
                                   (4992, 2048, 64)])   # 312 tiles: last wave 16/148 -> stream-K
@pytest.mark.parametrize("precision", [0, 1, 2])
def test_gemm(cuda, m, n, k, precision):
    import torch

    g = torch.Generator(device=cuda).manual_seed(m * n + k)
    a = torch.rand(m, k, device=cuda, generator=g) * 2 - 1
    b = torch.rand(k, n, device=cuda, generator=g) * 2 - 1
    want = a.double() @ b.double()
    got = lcnn.gemm(a.reshape(-1), b.reshape(-1), m, n, k, precision).view(m, n).double()
    err = (got - want).abs()
    bound = a.abs().double() @ b.abs().double()
    assert bool((err <= tolerance(precision, got, want, bound)).all()), float(err.max())


def test_fc_identity_and_hand_product(cuda):
    """test_softmax.cpp:156-190: identity weights are exact, [1 2]x[3;4] = 11."""
    import torch

    x = torch.from_numpy(rng_uniform(9, 24, -5, 5)).to(cuda)
    eye = torch.eye(6, device=cuda).reshape(-1)
    assert torch.equal(lcnn.gemm(x, eye, 4, 6, 6, lcnn.FP32), x)
    a = torch.tensor([1.0, 2.0], device=cuda)
    b = torch.tensor([3.0, 4.0], device=cuda)
    for prec in (0, 1, 2):
        assert float(lcnn.gemm(a, b, 1, 1, 2, prec)[0]) == 11.0


@pytest.mark.parametrize("m,n,k", [(128, 4096, 9216), (128, 4096, 4096), (128, 1000, 4096),
                                   (64, 1000, 4096), (256, 300, 96), (8, 37, 20), (132, 257, 36)])
@pytest.mark.parametrize("precision", [0, 1])
def test_fc_packed(cuda, m, n, k, precision):
    """fc on packed weights (lcnn_fc_pack_weights + lcnn_fc_forward_packed),
    x as NCHW rows [m][k] and as a CHWN producer [k][m]: same tolerances as
    the GEMM (the operand bits are identical, only the load path differs)."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(m + n * k)
    a = torch.rand(m, k, device=cuda, generator=g) * 2 - 1
    w = torch.rand(k, n, device=cuda, generator=g) * 2 - 1
    want = a.double() @ w.double()
    bound = a.abs().double() @ w.abs().double()
    packed = lcnn.pack_fc_weights(w.reshape(-1), k, n, precision)
    for layout, x in ((NCHW, a.contiguous()), (CHWN, a.t().contiguous())):
        if layout == CHWN and m % 4:
            continue
        got = lcnn.fc_forward_packed(x.reshape(-1), layout, packed, m, n, k, precision)
        got = got.view(m, n).double()
        err = (got - want).abs()
        assert bool((err <= tolerance(precision, got, want, bound)).all()), \
            (layout, float(err.max()))


def test_fc_packed_rejects_fp32(cuda):
    import torch

    w = torch.zeros(64, device=cuda)
    with pytest.raises(ValueError):
        lcnn.pack_fc_weights(w, 8, 8, lcnn.FP32)


def test_fc_packed_sync_words_zero_in_kernel(cuda):
    """lcnn_fc_forward_packed_ex: with caller-owned sync words the stream-K
    output is zeroed inside the fc kernel (no zeroing launch).  The output
    starts as NaN, so any element the kernel failed to zero before adding
    fragments stays NaN; one set of words serves launches of different grid
    sizes in a row and is left zero after each."""
    import torch

    from paper_1610_03618_b200 import capi

    sync = torch.zeros(capi.SYNC_BYTES // 8, dtype=torch.int64, device=cuda)
    for rep, (m, n, k) in enumerate([(128, 4096, 9216), (128, 4096, 4096), (256, 300, 96),
                                     (132, 257, 36), (128, 4096, 9216)]):
        g = torch.Generator(device=cuda).manual_seed(rep)
        a = torch.rand(m, k, device=cuda, generator=g) * 2 - 1
        w = torch.rand(k, n, device=cuda, generator=g) * 2 - 1
        want = a.double() @ w.double()
        bound = a.abs().double() @ w.abs().double()
        packed = lcnn.pack_fc_weights(w.reshape(-1), k, n, lcnn.TF32)
        for layout, x in ((NCHW, a.contiguous()), (CHWN, a.t().contiguous())):
            if layout == CHWN and m % 4:
                continue
            out = torch.full((m * n,), float("nan"), device=cuda)
            got = lcnn.fc_forward_packed(x.reshape(-1), layout, packed, m, n, k, lcnn.TF32,
                                         out=out, sync=sync).view(m, n).double()
            err = (got - want).abs()
            assert bool((err <= tolerance(lcnn.TF32, got, want, bound)).all()), \
                (m, n, k, layout, float(err.nan_to_num(1e30).max()))
            torch.cuda.synchronize()
            assert int(sync.abs().sum()) == 0, sync.tolist()


@pytest.mark.parametrize("case", [c for c in CASES if c[0] % 32 == 0])
def test_conv_packed_sync_words_zero_in_kernel(cuda, case):
    """lcnn_conv_forward_packed_ex on every CHWN route: the persistent
    kernel's stream-K output region is zeroed in-kernel (NaN-filled output
    before the launch), routes without in-kernel zeroing still launch the
    zeroing kernel; the sync words end zero."""
    import torch

    from paper_1610_03618_b200 import capi

    n, ci, h, w, co, f, stride, pad = case
    g = torch.Generator(device=cuda).manual_seed(sum(case))
    x = torch.rand(n, ci, h, w, device=cuda, generator=g) * 2 - 1
    filt = torch.rand(co, ci, f, f, device=cuda, generator=g) * 2 - 1
    want = _torch_conv64(x, filt, stride, pad)
    bound = _torch_conv64(x.abs(), filt.abs(), stride, pad)
    t = lcnn.DeviceTensor4D(n, ci, h, w, CHWN, x.permute(1, 2, 3, 0).contiguous().reshape(-1))
    packed = lcnn.pack_conv_filters(t, filt.contiguous(), co, f, f, stride, pad, lcnn.TF32)
    ho, wo = want.shape[2], want.shape[3]
    sync = torch.zeros(capi.SYNC_BYTES // 8, dtype=torch.int64, device=cuda)
    for _ in range(2):
        out = lcnn.DeviceTensor4D(n, co, ho, wo, CHWN,
                                  torch.full((n * co * ho * wo,), float("nan"), device=cuda))
        lcnn.conv_forward_packed(t, packed, co, f, f, stride, pad, lcnn.TF32, out=out, sync=sync)
        got = out.data.view(co, ho, wo, n).permute(3, 0, 1, 2).double()
        err = (got - want).abs()
        assert bool((err <= tolerance(lcnn.TF32, got, want, bound)).all()), \
            (case, float(err.nan_to_num(1e30).max()))
        torch.cuda.synchronize()
        assert int(sync.abs().sum()) == 0, sync.tolist()


def test_fc_packed_next_layer_prefetch_keeps_results(cuda):
    """lcnn_fc_forward_packed_ex with the next layer's packed weights as an L2
    prefetch target: the prefetch only warms L2, the product is unchanged
    (same tolerance as the plain call), for an fc6/fc7-shaped pair."""
    import torch

    g = torch.Generator(device=cuda).manual_seed(21)
    m, k, n, n2 = 128, 4096, 4096, 1000
    a = torch.rand(m, k, device=cuda, generator=g) * 2 - 1
    w = torch.rand(k, n, device=cuda, generator=g) * 2 - 1
    w2 = torch.rand(n, n2, device=cuda, generator=g) * 2 - 1
    pk = lcnn.pack_fc_weights(w.reshape(-1), k, n, lcnn.TF32)
    pk2 = lcnn.pack_fc_weights(w2.reshape(-1), n, n2, lcnn.TF32)
    want = a.double() @ w.double()
    bound = a.abs().double() @ w.abs().double()
    got = lcnn.fc_forward_packed(a.reshape(-1), NCHW, pk, m, n, k, lcnn.TF32,
                                 next_packed=pk2).view(m, n).double()
    assert bool(((got - want).abs() <= tolerance(lcnn.TF32, got, want, bound)).all())
