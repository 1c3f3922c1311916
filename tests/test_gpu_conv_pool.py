"""GPU parity for the fused convolution -> max pooling kernel
(lcnn_conv_maxpool_packed, csrc/conv.cu SharePoolOut): the reference runs the
two layers one after the other (run_network, net.cpp:284-353: conv_direct,
then pool_coarsened / pool_layout), so the fused kernel must return exactly
the bits of conv_forward_packed followed by pool_layout (max) -- every conv
value is the same K-ordered tensor-core sum, and the pooling keeps the
reference's compare-select tap order (pool.cpp:120).  Bit-exact (torch.equal),
including NaN / +-0 patterns in the input.  The unfused conv itself is held to
the TF32 bound against fp64 in test_gpu_conv_gemm.py.

Bit-exactness against the two-layer run needs the unfused conv to sum each
output whole: layers with at least a 60 %-full last wave of tiles (AlexNet
conv1 at any batch of 32k images) run whole tiles; small layers put their
tail on stream-K, whose fp32 fragments are added in another order, so there
the fused output is held to the conv's TF32 bound instead (max pooling is
1-Lipschitz: |max a - max b| <= max |a - b|, so the pooled bound is the
max-pooled per-output bound).
"""
import pytest

from oracle.oracle import CHWN
from paper_1610_03618_b200 import lcnn

pytestmark = pytest.mark.gpu

# (n, c_i, h, w, c_o, f, stride, pad, pool window, pool stride)
EXACT = [
    (128, 3, 227, 227, 96, 11, 4, 0, 3, 2),  # AlexNet conv1 -> pool1, as benched
    (32, 3, 227, 227, 96, 11, 4, 0, 3, 2),   # one 32-image group (strong-scaled shard)
    (64, 3, 100, 100, 96, 11, 4, 0, 3, 2),   # 23x23 conv -> 11x11 (last strip partial)
]
CASES = EXACT + [
    (32, 3, 67, 71, 40, 11, 4, 2, 3, 2),     # padding, c_o = 40 (one real channel warp + part)
    (32, 3, 64, 64, 64, 7, 2, 3, 3, 2),      # 32x32 conv -> 15x15
    (32, 3, 64, 64, 64, 5, 1, 2, 3, 2),      # stride-1 conv, 64x64 -> 31x31
    (64, 3, 96, 96, 96, 11, 4, 0, 2, 2),     # 22x22 conv -> 11x11 with 2x2 windows
    (32, 1, 45, 45, 128, 5, 2, 0, 2, 2),     # c_o = 128, odd conv extent (21 -> 10)
]
# TAPS row-pair layers (C_o <= 64, channel planes >= 4 MB) with a 2x2 pool:
# the pool runs in the row-pair epilogue (TapsParams::pool); >= 8 waves of
# whole tiles, so the unfused conv sums every output whole -> bit-exact
TAPS = [
    (32, 32, 193, 185, 48, 3, 1, 1, 2, 2),   # odd extents: last row pair / pixel block partial, c_o 48
    (64, 32, 128, 160, 64, 3, 1, 1, 2, 2),   # two image groups
    (32, 32, 182, 182, 128, 3, 1, 1, 2, 2),  # C_o 128: two-accumulator row pairs
    (64, 64, 129, 131, 160, 3, 1, 1, 2, 2),  # two accumulators, odd extents, 2 channel tiles
]
EXACT += TAPS
CASES += TAPS


def _run(cuda, case, seed=0, special=False):
    import torch

    n, ci, h, w, co, f, s, p, pw, ps = case
    g = torch.Generator(device=cuda).manual_seed(seed)
    x = (torch.rand(ci, h, w, n, device=cuda, generator=g) * 2 - 1).reshape(-1)
    filt = (torch.rand(co, ci, f, f, device=cuda, generator=g) * 2 - 1).contiguous()
    if special:
        # signed zeros and exact ties: zero filters for some channels (every
        # conv output of those channels is a zero, so the pool keeps its
        # first tap), signed-zero inputs elsewhere.  (Non-finite inputs are
        # not compared: SHARE reads neighbouring pixels into zero-weight K
        # padding rows, and 0 x NaN contaminates outputs by tile position,
        # which differs between the 8-pixel and the 7-pixel tiling; DESIGN 8.)
        idx = torch.randint(0, x.numel(), (4096,), device=cuda, generator=g)
        x[idx[:2048]] = 0.0
        x[idx[2048:]] = -0.0
        filt[::7] = 0.0
        filt[1::11] = -0.0
    t = lcnn.DeviceTensor4D(n, ci, h, w, CHWN, x)
    assert lcnn.conv_maxpool_supported(t, co, f, f, s, p, lcnn.TF32, pw, ps), case
    packed = lcnn.pack_conv_filters(t, filt, co, f, f, s, p, lcnn.TF32)
    conv = lcnn.conv_forward_packed(t, packed, co, f, f, s, p, lcnn.TF32)
    want, _ = lcnn.pool_layout(conv, lcnn.PoolParams(pw, pw, ps, lcnn.MAX))
    got = lcnn.conv_maxpool_packed(t, packed, co, f, f, s, p, lcnn.TF32, pw, ps)
    torch.cuda.synchronize()
    assert (got.n, got.c, got.h, got.w) == (want.n, want.c, want.h, want.w)
    if case in EXACT:
        a, b = got.data.view(torch.int32), want.data.view(torch.int32)
        bad = int((a != b).sum())
        assert bad == 0, (case, bad, got.data.numel())
    if special:  # non-finite inputs: the unfused SHARE route is the reference (DESIGN 8)
        assert case in EXACT
        return got
    # against fp64: conv64 -> max pool, with the max-pooled TF32 bound
    xn = x.view(ci, h, w, n).permute(3, 0, 1, 2).double()
    conv64 = torch.nn.functional.conv2d(xn, filt.double(), stride=s, padding=p)
    bound = torch.nn.functional.conv2d(xn.abs().nan_to_num(0.0), filt.double().abs(), stride=s,
                                       padding=p)
    ref = torch.nn.functional.max_pool2d(conv64, pw, ps)
    tol = torch.nn.functional.max_pool2d(bound, pw, ps) * 2.0 ** -9 + 1e-6
    g = got.data.view(co, got.h, got.w, n).permute(3, 0, 1, 2).double()
    finite = torch.isfinite(ref)
    assert bool((torch.isfinite(g) == finite).all()), case
    err = (g - ref).abs()[finite]
    assert bool((err <= tol[finite]).all()), (case, float(err.max()))
    return got


@pytest.mark.parametrize("case", CASES)
def test_conv_maxpool_fused_bit_exact(cuda, case):
    _run(cuda, case)


def test_conv_maxpool_fused_special_values(cuda):
    _run(cuda, EXACT[1], seed=3, special=True)


def test_conv_maxpool_fused_repeatable(cuda):
    import torch

    a = _run(cuda, CASES[1], seed=5)
    b = _run(cuda, CASES[1], seed=5)
    assert torch.equal(a.data.view(torch.int32), b.data.view(torch.int32))


def test_conv_maxpool_unsupported_pairs(cuda):
    import torch

    x = torch.zeros(32 * 64 * 28 * 28, device=cuda)
    t = lcnn.DeviceTensor4D(32, 64, 28, 28, CHWN, x)
    # a CI-routed 3x3 layer, a stride-1 pool, FP32: not covered -> callers run two layers
    assert not lcnn.conv_maxpool_supported(t, 64, 3, 3, 1, 1, lcnn.TF32, 2, 2)
    x3 = torch.zeros(32 * 3 * 67 * 67, device=cuda)
    t3 = lcnn.DeviceTensor4D(32, 3, 67, 67, CHWN, x3)
    assert not lcnn.conv_maxpool_supported(t3, 96, 11, 11, 4, 0, lcnn.TF32, 3, 1)
    assert not lcnn.conv_maxpool_supported(t3, 96, 11, 11, 4, 0, lcnn.FP32, 3, 2)
    with pytest.raises(Exception):
        lcnn.conv_maxpool_packed(t, torch.zeros(1 << 20, dtype=torch.uint8, device=cuda),
                                 64, 3, 3, 1, 1, lcnn.TF32, 2, 2)


def test_conv_maxpool_taps_vgg_conv1_2_full_size(cuda):
    """VGG-16 conv1_2 -> pool1 exactly as the VGG-16 forward runs it (128
    images, 64 -> 64 channels, 224 x 224, 3 x 3 pad 1, then 2 x 2 / 2 max):
    bit-equal to the two-layer run (the fp64 bound is checked on the smaller
    TAPS cases; an fp64 conv of this size takes minutes)."""
    import torch

    n, ci, h, w, co = 128, 64, 224, 224, 64
    g = torch.Generator(device=cuda).manual_seed(11)
    x = (torch.rand(ci * h * w * n, device=cuda, generator=g) * 2 - 1)
    filt = (torch.rand(co, ci, 3, 3, device=cuda, generator=g) * 2 - 1).contiguous()
    t = lcnn.DeviceTensor4D(n, ci, h, w, CHWN, x)
    assert lcnn.conv_maxpool_supported(t, co, 3, 3, 1, 1, lcnn.TF32, 2, 2)
    packed = lcnn.pack_conv_filters(t, filt, co, 3, 3, 1, 1, lcnn.TF32)
    conv = lcnn.conv_forward_packed(t, packed, co, 3, 3, 1, 1, lcnn.TF32)
    want, _ = lcnn.pool_layout(conv, lcnn.PoolParams(2, 2, 2, lcnn.MAX))
    del conv
    got = lcnn.conv_maxpool_packed(t, packed, co, 3, 3, 1, 1, lcnn.TF32, 2, 2)
    torch.cuda.synchronize()
    assert (got.n, got.c, got.h, got.w) == (n, co, 112, 112)
    assert torch.equal(got.data.view(torch.int32), want.data.view(torch.int32))


def test_conv_maxpool_taps_special_values(cuda):
    _run(cuda, TAPS[0], seed=4, special=True)


def test_conv_maxpool_taps_vgg_conv2_2_full_size(cuda):
    """VGG-16 conv2_2 -> pool2 as the forward runs it (128 images, 128 -> 128
    channels, 112 x 112): bit-equal to the two-layer run."""
    import torch

    n, ci, h, w, co = 128, 128, 112, 112, 128
    g = torch.Generator(device=cuda).manual_seed(12)
    x = (torch.rand(ci * h * w * n, device=cuda, generator=g) * 2 - 1)
    filt = (torch.rand(co, ci, 3, 3, device=cuda, generator=g) * 2 - 1).contiguous()
    t = lcnn.DeviceTensor4D(n, ci, h, w, CHWN, x)
    assert lcnn.conv_maxpool_supported(t, co, 3, 3, 1, 1, lcnn.TF32, 2, 2)
    packed = lcnn.pack_conv_filters(t, filt, co, 3, 3, 1, 1, lcnn.TF32)
    conv = lcnn.conv_forward_packed(t, packed, co, 3, 3, 1, 1, lcnn.TF32)
    want, _ = lcnn.pool_layout(conv, lcnn.PoolParams(2, 2, 2, lcnn.MAX))
    del conv
    got = lcnn.conv_maxpool_packed(t, packed, co, 3, 3, 1, 1, lcnn.TF32, 2, 2)
    torch.cuda.synchronize()
    assert (got.n, got.c, got.h, got.w) == (n, co, 56, 56)
    assert torch.equal(got.data.view(torch.int32), want.data.view(torch.int32))


def _to_blocked(t, n, c, h, w):
    """CHWN [c][h][w][n] -> the blocked [n/32][h][w][c][32] (flat)."""
    return t.view(c, h, w, n // 32, 32).permute(3, 1, 2, 0, 4).contiguous().view(-1)


def _from_blocked(t, n, c, h, w):
    return t.view(n // 32, h, w, c, 32).permute(3, 1, 2, 0, 4).contiguous().view(-1)


def test_hwcn32_vgg_conv1_1_to_conv1_2_pool1_full_size(cuda):
    """The run_network-internal blocked activation between VGG conv1_1 (ROW row
    pairs, quad-box epilogue writing [N/32][H][W][C][32]) and conv1_2 + pool1
    (TAPS row pairs reading it as 4 KB runs): the producer writes the same
    values as the CHWN route, permuted (fp32 stream-K fragments may add in
    another order: 1e-6 relative), and the consumer returns exactly the bits
    of the CHWN conv1_2 + pool1 on the same values."""
    import torch

    n, h, w = 128, 224, 224
    g = torch.Generator(device=cuda).manual_seed(5)
    x = torch.rand(3 * h * w * n, device=cuda, generator=g) * 2 - 1
    f1 = (torch.rand(64, 3, 3, 3, device=cuda, generator=g) * 2 - 1).contiguous()
    f2 = (torch.rand(64, 64, 3, 3, device=cuda, generator=g) * 0.2 - 0.1).contiguous()
    t = lcnn.DeviceTensor4D(n, 3, h, w, CHWN, x)
    assert lcnn.conv_hwcn32_supported(t, 64, 3, 3, 1, 1, lcnn.TF32, 0, 0, lcnn.OUT_HWCN32)
    assert not lcnn.conv_hwcn32_supported(t, 64, 3, 3, 1, 1, lcnn.TF32, 0, 0, lcnn.IN_HWCN32)
    assert not lcnn.conv_hwcn32_supported(t, 64, 3, 3, 1, 1, lcnn.FP32, 0, 0, lcnn.OUT_HWCN32)
    p1 = lcnn.pack_conv_filters(t, f1, 64, 3, 3, 1, 1, lcnn.TF32)
    c11 = lcnn.conv_forward_packed(t, p1, 64, 3, 3, 1, 1, lcnn.TF32)
    c11b = lcnn.conv_forward_packed(t, p1, 64, 3, 3, 1, 1, lcnn.TF32, blk=lcnn.OUT_HWCN32)
    torch.cuda.synchronize()
    ref = _to_blocked(c11.data, n, 64, h, w)
    scale = ref.abs().max().item()
    assert (c11b.data - ref).abs().max().item() <= 1e-6 * scale
    del c11, ref
    assert lcnn.conv_hwcn32_supported(c11b, 64, 3, 3, 1, 1, lcnn.TF32, 2, 2, lcnn.IN_HWCN32)
    p2 = lcnn.pack_conv_filters(c11b, f2, 64, 3, 3, 1, 1, lcnn.TF32)
    got = lcnn.conv_maxpool_packed(c11b, p2, 64, 3, 3, 1, 1, lcnn.TF32, 2, 2,
                                   blk=lcnn.IN_HWCN32)
    plain = lcnn.DeviceTensor4D(n, 64, h, w, CHWN, _from_blocked(c11b.data, n, 64, h, w))
    want = lcnn.conv_maxpool_packed(plain, p2, 64, 3, 3, 1, 1, lcnn.TF32, 2, 2)
    torch.cuda.synchronize()
    assert (got.n, got.c, got.h, got.w) == (n, 64, 112, 112)
    assert torch.equal(got.data.view(torch.int32), want.data.view(torch.int32))


def test_hwcn32_unsupported_routes_fail_loudly(cuda):
    """A blocked flag on a route that cannot honour it is an error, never a
    silent CHWN run (AlexNet conv1 SHARE route; a pool-fused SHARE consumer)."""
    import torch

    from paper_1610_03618_b200 import errors

    n = 32
    x = torch.rand(3 * 227 * 227 * n, device=cuda)
    f = torch.rand(96, 3, 11, 11, device=cuda).contiguous()
    t = lcnn.DeviceTensor4D(n, 3, 227, 227, CHWN, x)
    assert not lcnn.conv_hwcn32_supported(t, 96, 11, 11, 4, 0, lcnn.TF32, 0, 0, lcnn.OUT_HWCN32)
    p = lcnn.pack_conv_filters(t, f, 96, 11, 11, 4, 0, lcnn.TF32)
    with pytest.raises(errors.Error):
        lcnn.conv_forward_packed(t, p, 96, 11, 11, 4, 0, lcnn.TF32, blk=lcnn.OUT_HWCN32)
    with pytest.raises(errors.Error):
        lcnn.conv_maxpool_packed(t, p, 96, 11, 11, 4, 0, lcnn.TF32, 3, 2, blk=lcnn.IN_HWCN32)
