"""GPU parity: CHWN<->NCHW transform kernel and the generic permute, through
the C ABI, bit-exact against the CPU oracle / the reference's fixtures."""
import numpy as np
import pytest

from oracle.oracle import CHWN, HWCN, NCHW, NHWC, C, bit_equal, rng_uniform
from paper_1610_03618_b200 import errors, lcnn

pytestmark = pytest.mark.gpu

# Table 1 fixture input dims (fixtures.cpp:59-93): (n, c, h, w)
FIXTURE_DIMS = {
    "CV1": (128, 1, 28, 28), "CV2": (128, 16, 14, 14), "PL1": (128, 16, 28, 28),
    "PL2": (128, 16, 14, 14), "CV3": (128, 3, 24, 24), "CV4": (128, 64, 12, 12),
    "PL3": (128, 64, 24, 24), "PL4": (128, 64, 12, 12), "PL5": (128, 96, 55, 55),
    "PL6": (128, 192, 27, 27), "PL7": (128, 256, 13, 13), "CV5": (64, 3, 224, 224),
    "CV6": (64, 96, 55, 55), "CV7": (64, 256, 13, 13), "CV8": (64, 384, 13, 13),
    "PL8": (64, 96, 110, 110), "PL9": (64, 256, 26, 26), "PL10": (64, 256, 13, 13),
    "CV9": (32, 3, 224, 224), "CV10": (32, 128, 56, 56), "CV11": (32, 256, 28, 28),
    "CV12": (32, 512, 14, 14), "CLASS1": (128, 10, 1, 1), "CLASS2": (128, 10, 1, 1),
    "CLASS3": (128, 1000, 1, 1), "CLASS4": (64, 1000, 1, 1), "CLASS5": (32, 1000, 1, 1),
}


def dev(x, dims, layout, device):
    return lcnn.DeviceTensor4D.from_host(x, *dims, layout, device=device)


def test_iota_kat(cuda, kats):
    k = kats["transform_iota"]
    t = dev(np.arange(16, dtype=np.float32), k["dims"], k["src_layout"], cuda)
    out = lcnn.transform(t, k["dst_layout"])
    assert out.to_host().tolist() == k["expected"]
    back = lcnn.transform(out, k["src_layout"])
    assert back.to_host().tolist() == list(range(16))


def test_reference_fixtures(cuda, ref_vectors):
    v = ref_vectors
    keys = sorted({k.split("_")[1] for k in v.files if k.startswith("transform_")}, key=int)
    assert len(keys) >= 30
    for k in keys:
        n, c, h, w, sl, dl = v[f"transform_{k}_meta"].tolist()
        t = dev(v[f"transform_{k}_in"], (n, c, h, w), sl, cuda)
        assert bit_equal(lcnn.transform(t, dl).to_host(), v[f"transform_{k}_out"]), (k, sl, dl)
        assert bit_equal(lcnn.transform_naive(t, dl).to_host(), v[f"transform_{k}_out"])


def test_plan_errors_raise(cuda, kats):
    n, c, h, w = kats["plan_errors"]["tensor"]["dims"]
    t = dev(rng_uniform(3, n * c * h * w, -100, 100), (n, c, h, w), CHWN, cuda)
    for case in kats["plan_errors"]["cases"]:
        plan = lcnn.TransformPlan(case["src"], case["dst"], case["tile"], case["wide"])
        with pytest.raises(errors.PlanError):
            lcnn.transform_tiled(t, case["dst"], plan)
    with pytest.raises(errors.PlanError):  # mismatched source layout
        lcnn.transform_tiled(t, CHWN, lcnn.make_plan(NCHW, CHWN, n, c, h, w))


def test_acceptance_criterion3_random_shapes(cuda):
    """acceptance.cpp:163-213: 200 random shapes, batches {1,3,16,64,96,128}."""
    rng = np.random.default_rng(42)
    batches = [1, 3, 16, 64, 96, 128]
    for trial in range(200):
        n = batches[trial % 6]
        c, h, w = (int(x) for x in rng.integers(1, 17, 3))
        x = rng_uniform(trial, n * c * h * w)
        src = dev(x, (n, c, h, w), CHWN, cuda)
        want = C.transform(x, n, c, h, w, CHWN, NCHW)
        plan = lcnn.make_plan(CHWN, NCHW, n, c, h, w)
        assert plan.wide_copy == (n >= 64)
        plan.wide_copy = False
        tiled = lcnn.transform_tiled(src, NCHW, plan)
        assert bit_equal(tiled.to_host(), want), (n, c, h, w)
        if n >= 64:
            plan.wide_copy = True
            assert bit_equal(lcnn.transform_tiled(src, NCHW, plan).to_host(), want)
        back = lcnn.transform_tiled(tiled, CHWN, lcnn.make_plan(NCHW, CHWN, n, c, h, w))
        assert bit_equal(back.to_host(), x)


def test_fixture_shapes_full_size(cuda):
    """All 27 Table-1 input shapes at full size, both directions, vs the C oracle."""
    for name, (n, c, h, w) in FIXTURE_DIMS.items():
        x = rng_uniform(hash(name) % 1000, n * c * h * w)
        for sl, dl in ((CHWN, NCHW), (NCHW, CHWN)):
            out = lcnn.transform(dev(x, (n, c, h, w), sl, cuda), dl).to_host()
            assert bit_equal(out, C.transform(x, n, c, h, w, sl, dl)), (name, sl)


def test_all_layout_pairs_compose(cuda):
    """test_layout.cpp:132-154: compositions collapse, chains return bit-identical."""
    n, c, h, w = 6, 4, 3, 5
    x = rng_uniform(23, n * c * h * w, -100, 100)
    t = dev(x, (n, c, h, w), NCHW, cuda)
    layouts = (NCHW, CHWN, NHWC, HWCN)
    for mid in layouts:
        for dst in layouts:
            via = lcnn.transform(lcnn.transform(t, mid), dst)
            assert bit_equal(via.to_host(), lcnn.transform(t, dst).to_host())
            assert bit_equal(via.to_host(), C.transform(x, n, c, h, w, NCHW, dst))
    cur = t
    for step in (CHWN, NHWC, HWCN, NCHW):
        cur = lcnn.transform(cur, step)
    assert bit_equal(cur.to_host(), x)


def test_config3_sweep_roundtrip(cuda):
    """Config 3 (AlexNet/VGG activations, N 32-256): size-independent check --
    the kernel equals torch's permute (pure data movement) and round-trips."""
    import torch

    shapes = [(3, 227, 227), (96, 55, 55), (256, 13, 13), (64, 112, 112), (512, 7, 7)]
    for n in (32, 256):
        for c, h, w in shapes:
            x = torch.randn(c * h * w * n, device=cuda)
            t = lcnn.DeviceTensor4D(n, c, h, w, CHWN, x)
            out = lcnn.transform(t, NCHW)
            want = x.view(c, h, w, n).permute(3, 0, 1, 2).contiguous().view(-1)
            assert torch.equal(out.data, want)
            back = lcnn.transform(out, CHWN)
            assert torch.equal(back.data, x)


def test_offset_pointers_and_odd_sizes(cuda):
    """Unaligned base pointers force the scalar paths; results stay exact."""
    import torch

    n, c, h, w = 64, 3, 5, 7
    x = rng_uniform(5, n * c * h * w + 1)
    buf = torch.from_numpy(x).to(cuda)
    t = lcnn.DeviceTensor4D(n, c, h, w, CHWN, buf[1:])
    out = lcnn.transform(t, NCHW)
    assert bit_equal(out.to_host(), C.transform(x[1:], n, c, h, w, CHWN, NCHW))


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 12, 16, 17, 32])
def test_small_batch_paths_bit_exact(cuda, n):
    """The short-side transpose (N <= 16 after sharding: contiguous runs both
    ways, 128-bit when aligned) and the N = 1 copy, both directions, on the
    AlexNet/VGG activation shapes of config 3 and on odd extents."""
    import torch

    for (c, h, w) in ((96, 55, 55), (3, 227, 227), (64, 56, 56), (7, 5, 3), (256, 6, 6)):
        x = rng_uniform(n * c + h, n * c * h * w)
        for src, dst in ((NCHW, CHWN), (CHWN, NCHW)):
            t = dev(x, (n, c, h, w), src, cuda)
            got = lcnn.transform(t, dst).to_host()
            assert bit_equal(got, C.transform(x, n, c, h, w, src, dst)), (n, c, h, w, src)
        # unaligned (4-byte offset) source: the scalar side of the kernel
        buf = torch.from_numpy(np.concatenate([np.zeros(1, np.float32), x])).to(cuda)
        t = lcnn.DeviceTensor4D(n, c, h, w, CHWN, buf[1:])
        got = lcnn.transform(t, NCHW).to_host()
        assert bit_equal(got, C.transform(x, n, c, h, w, CHWN, NCHW)), (n, c, h, w, "unaligned")


@pytest.mark.parametrize("dims", [(8, 96, 27, 27), (33, 5, 7, 41), (1, 3, 224, 224), (64, 64, 14, 14)])
def test_all_layout_pairs_bit_exact(cuda, dims):
    """transform_naive (layout.cpp:77-97) for all 12 ordered pairs of the four
    layouts: the tiled batched-transpose kernel (innermost dims differ) and
    the run-copy kernel (CHWN<->HWCN share N innermost), against the oracle."""
    n, c, h, w = dims
    x = rng_uniform(sum(dims), n * c * h * w)
    for src in (NCHW, CHWN, NHWC, HWCN):
        t = dev(x, dims, src, cuda)
        for dst in (NCHW, CHWN, NHWC, HWCN):
            if dst == src:
                continue
            got = lcnn.transform_naive(t, dst).to_host()
            assert bit_equal(got, C.transform(x, n, c, h, w, src, dst)), (dims, src, dst)
