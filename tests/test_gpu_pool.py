"""GPU parity: max/avg pooling kernels (CHWN, NCHW, coarsened) through the C
ABI against the CPU oracle and the reference's fixtures.  Max is bit-exact by
construction; average reproduces the reference's fp32 operation order and is
checked bit-exact too (the 1e-6 approx_equal bar of bench.cpp:114 is the
documented tolerance)."""
import numpy as np
import pytest

from oracle.oracle import CHWN, NCHW, NHWC, C, approx_equal, bit_equal, rng_uniform
from paper_1610_03618_b200 import capi, errors, lcnn

pytestmark = pytest.mark.gpu


def dev(x, dims, layout, device):
    return lcnn.DeviceTensor4D.from_host(x, *dims, layout, device=device)


def P(wh, ww, s, avg):
    return lcnn.PoolParams(wh, ww, s, lcnn.AVERAGE if avg else lcnn.MAX)


def test_kats(cuda, kats):
    x = np.arange(1, 13, dtype=np.float32)
    for layout in (NCHW, CHWN):
        out, rep = lcnn.pool_layout(dev(x, (1, 1, 1, 12), layout, cuda), P(1, 4, 2, True))
        assert out.to_host().tolist() == kats["pool_line_average"]["expected"]
        k = kats["pool_line_accounting"]
        assert rep.as_tuple() == (k["input_loads"], k["output_stores"], k["distinct_inputs"])
    x = np.arange(1, 17, dtype=np.float32)
    for layout in (NCHW, CHWN):
        out, _ = lcnn.pool_layout(dev(x, (1, 1, 4, 4), layout, cuda), P(2, 2, 2, False))
        assert out.to_host().tolist() == kats["pool_ramp_max"]["expected"]
    with pytest.raises(errors.ShapeError):
        lcnn.pool_layout(dev(np.zeros(9, np.float32), (1, 1, 3, 3), NCHW, cuda), P(4, 4, 1, False))
    k = kats["pool_coarsened_loads"]
    x = rng_uniform(8, 33, -10, 10)
    t = dev(x, (1, 1, 3, 11), CHWN, cuda)
    out, rep = lcnn.pool_coarsened(t, P(3, 3, 2, False), lcnn.CoarseningPlan(1, 2))
    assert out.w == k["w_out"] and rep.input_loads == k["coarsened_loads"]
    _, plain = lcnn.pool_layout(t, P(3, 3, 2, False))
    assert plain.input_loads == k["plain_loads"]
    for case in kats["pool_plan_errors"]["cases"]:
        tt = dev(np.zeros(256, np.float32), (2, 2, 8, 8), case["layout"], cuda)
        with pytest.raises({"PlanError": errors.PlanError, "LayoutError": errors.LayoutError}[case["error"]]):
            lcnn.pool_coarsened(tt, P(2, 2, 2, False), lcnn.CoarseningPlan(*case["plan"]))
    with pytest.raises(errors.LayoutError):
        lcnn.pool_layout(dev(np.zeros(64, np.float32), (2, 2, 4, 4), NHWC, cuda), P(2, 2, 2, False))


def test_reference_fixtures(cuda, ref_vectors):
    v = ref_vectors
    keys = sorted({k.split("_")[1] for k in v.files if k.startswith("pool_")}, key=int)
    for k in keys:
        n, c, h, w, layout, wh, ww, s, avg = v[f"pool_{k}_meta"].tolist()
        t = dev(v[f"pool_{k}_in"], (n, c, h, w), layout, cuda)
        out, rep = lcnn.pool_layout(t, P(wh, ww, s, avg))
        assert bit_equal(out.to_host(), v[f"pool_{k}_out"]), (k, layout, wh, s, avg)
        assert rep.as_tuple() == tuple(v[f"pool_{k}_report"].tolist())
        assert bit_equal(lcnn.pool_oracle(t, P(wh, ww, s, avg)).to_host(), v[f"pool_{k}_oracle"])
        if layout == CHWN:
            for fh, fw in ((2, 2), (1, 3), (3, 1), (4, 4)):
                o2, r2 = lcnn.pool_coarsened(t, P(wh, ww, s, avg), lcnn.CoarseningPlan(fh, fw))
                assert bit_equal(o2.to_host(), v[f"pool_{k}_coarse_{fh}x{fw}_out"]), (k, fh, fw)
                assert r2.as_tuple() == tuple(v[f"pool_{k}_coarse_{fh}x{fw}_report"].tolist())


def test_random_trials_vs_oracle(cuda):
    """test_pool.cpp:109-128 recipe, widened to both modes, all kernels."""
    rng = np.random.default_rng(6)
    for trial in range(60):
        h = int(rng.integers(4, 17))
        w = int(rng.integers(4, 17))
        win, stride = 2 + trial % 2, 1 + trial % 3
        avg = bool(trial % 2)
        n, c = (int(x) for x in rng.integers(1, 17, 2))
        x = rng_uniform(trial, n * c * h * w, -10, 10)
        base = dev(x, (n, c, h, w), NCHW, cuda)
        want_nchw, _ = C.pool_plain(x, n, c, h, w, NCHW, win, win, stride, avg)
        got, _ = lcnn.pool_layout(base, P(win, win, stride, avg))
        assert bit_equal(got.to_host(), want_nchw), (trial, n, c, h, w)
        xc = C.transform(x, n, c, h, w, NCHW, CHWN)
        chwn = dev(xc, (n, c, h, w), CHWN, cuda)
        want_chwn, _ = C.pool_plain(xc, n, c, h, w, CHWN, win, win, stride, avg)
        got, _ = lcnn.pool_layout(chwn, P(win, win, stride, avg))
        assert bit_equal(got.to_host(), want_chwn)
        for fh, fw in ((2, 2), (1, 4), (3, 2), (5, 1)):
            got, _ = lcnn.pool_coarsened(chwn, P(win, win, stride, avg), lcnn.CoarseningPlan(fh, fw))
            assert bit_equal(got.to_host(), want_chwn), (trial, fh, fw)
        for fh, fw in ((2, 1), (4, 1), (3, 2), (1, 2), (6, 1)):
            got, _ = lcnn.pool_coarsened_nchw(base, P(win, win, stride, avg), lcnn.CoarseningPlan(fh, fw))
            assert bit_equal(got.to_host(), want_nchw), (trial, fh, fw)
        # cross-layout agreement with the fp64 oracle at the reference's tolerance
        oracle = C.pool_oracle(x, n, c, h, w, NCHW, win, win, stride, avg)
        assert approx_equal(want_nchw, oracle, 1e-6 if avg else 0.0)


def test_acceptance_criterion4_every_plan(cuda):
    """acceptance.cpp:217-241: every (fh, fw) up to the cap on 3x4x24x24."""
    n, c, h, w = 3, 4, 24, 24
    x = rng_uniform(4, n * c * h * w)
    t = dev(x, (n, c, h, w), CHWN, cuda)
    for avg in (False, True):
        want, _ = C.pool_plain(x, n, c, h, w, CHWN, 3, 3, 2, avg)
        plans = 0
        for fh in range(1, 65):
            for fw in range(1, 65 // fh + 1):
                if fh * fw > 64:
                    continue
                got, rep = lcnn.pool_coarsened(t, P(3, 3, 2, avg), lcnn.CoarseningPlan(fh, fw))
                assert bit_equal(got.to_host(), want), (fh, fw, avg)
                _, crep = C.pool_coarsened(x, n, c, h, w, CHWN, 3, 3, 2, avg, fh, fw)
                assert rep.as_tuple() == crep
                plans += 1
        assert plans == 280


def test_pool_fixtures_full_size(cuda):
    """PL1..PL10 at full size (fixtures.cpp:59-93), both layouts, max + avg."""
    fixtures = {"PL1": (128, 16, 28, 2, 2), "PL2": (128, 16, 14, 2, 2), "PL3": (128, 64, 24, 3, 2),
                "PL4": (128, 64, 12, 3, 2), "PL5": (128, 96, 55, 3, 2), "PL6": (128, 192, 27, 3, 2),
                "PL7": (128, 256, 13, 3, 2), "PL8": (64, 96, 110, 3, 2), "PL9": (64, 256, 26, 3, 2),
                "PL10": (64, 256, 13, 3, 2)}
    for name, (n, c, hw, win, s) in fixtures.items():
        x = rng_uniform(len(name), n * c * hw * hw)
        for avg in (False, True):
            for layout in (CHWN, NCHW):
                xin = x if layout == NCHW else C.transform(x, n, c, hw, hw, NCHW, CHWN)
                t = dev(xin, (n, c, hw, hw), layout, cuda)
                want, _ = C.pool_plain(xin, n, c, hw, hw, layout, win, win, s, avg)
                got, _ = lcnn.pool_layout(t, P(win, win, s, avg))
                assert bit_equal(got.to_host(), want), (name, layout, avg)
                if layout == NCHW:  # the pipelined kernel's 2-wide output blocks at full size
                    for fh, fw in ((3, 2), (2, 2), (4, 2)):
                        got, _ = lcnn.pool_coarsened_nchw(t, P(win, win, s, avg),
                                                          lcnn.CoarseningPlan(fh, fw))
                        assert bit_equal(got.to_host(), want), (name, fh, fw, avg)
                if layout == CHWN:
                    got, rep = lcnn.pool_coarsened(t, P(win, win, s, avg), lcnn.CoarseningPlan(2, 2))
                    assert bit_equal(got.to_host(), want)
                    if s < win:  # acceptance.cpp:489-503: coarsening strictly saves loads
                        _, plain = lcnn.pool_layout(t, P(win, win, s, avg))
                        assert rep.input_loads < plain.input_loads


def test_vgg_pools_batch_independence(cuda):
    """Config 4 shapes at N=256 (sharded 1/2/4/8) -- size-independent checks:
    the N-shards pooled separately concatenate to the unsharded result, and the
    CHWN/NCHW kernels agree through the transform kernel."""
    import torch

    for c, hw in ((512, 14), (256, 56), (64, 224)):
        n = 256
        x = torch.rand(n * c * hw * hw, device=cuda) * 2 - 1
        full = lcnn.DeviceTensor4D(n, c, hw, hw, NCHW, x)
        out_full, _ = lcnn.pool_layout(full, P(2, 2, 2, False))
        ref = torch.nn.functional.max_pool2d(x.view(n, c, hw, hw), 2, 2).reshape(-1)
        assert torch.equal(out_full.data, ref)  # max pooling: exact for any order
        chwn = lcnn.transform(full, CHWN)
        out_c, _ = lcnn.pool_coarsened(chwn, P(2, 2, 2, False), lcnn.CoarseningPlan(2, 2))
        assert torch.equal(lcnn.transform(out_c, NCHW).data, out_full.data)
        for g in (2, 4, 8):
            shards = []
            for r in range(g):
                xs = x.view(n, -1)[r * n // g:(r + 1) * n // g].reshape(-1)
                o, _ = lcnn.pool_layout(lcnn.DeviceTensor4D(n // g, c, hw, hw, NCHW, xs), P(2, 2, 2, False))
                shards.append(o.data)
            assert torch.equal(torch.cat(shards), out_full.data)
        del x, full, out_full, chwn, out_c, ref
        torch.cuda.empty_cache()


def test_unaligned_and_odd_batches(cuda):
    import torch

    for n in (1, 3, 5, 17):
        c, h, w = 3, 11, 9
        x = rng_uniform(n, n * c * h * w + 1)
        buf = torch.from_numpy(x).to(cuda)
        for layout in (CHWN, NCHW):
            t = lcnn.DeviceTensor4D(n, c, h, w, layout, buf[1:])
            want, _ = C.pool_plain(x[1:], n, c, h, w, layout, 3, 3, 2, True)
            got, _ = lcnn.pool_layout(t, P(3, 3, 2, True))
            assert bit_equal(got.to_host(), want), (n, layout)


def test_window_equals_image_and_generic_windows(cuda):
    for (h, w, wh, ww, s) in ((5, 5, 5, 5, 1), (7, 9, 2, 4, 3), (12, 12, 4, 4, 4), (6, 6, 1, 1, 1)):
        n, c = 8, 3
        x = rng_uniform(h * w, n * c * h * w)
        for layout in (CHWN, NCHW):
            for avg in (False, True):
                t = dev(x, (n, c, h, w), layout, cuda)
                want, _ = C.pool_plain(x, n, c, h, w, layout, wh, ww, s, avg)
                got, _ = lcnn.pool_layout(t, P(wh, ww, s, avg))
                assert bit_equal(got.to_host(), want), (h, w, wh, ww, s, layout, avg)


def test_pool_tuner_plans_are_cached_and_bit_exact(cuda):
    """lcnn_pool_tune measures the layout's kernel plans on the shape, caches
    the fastest (lookup returns it, pool_layout then runs it), and any plan it
    can return gives the plain kernel's bits (PAPER.md:227 autotuning;
    pool.cpp:272-331 is the reference's hill climb over the same space)."""
    for layout, (n, c, h, win, s) in ((CHWN, (64, 32, 56, 2, 2)), (NCHW, (16, 24, 55, 3, 2)),
                                      (NCHW, (8, 16, 112, 2, 2)), (CHWN, (32, 16, 27, 3, 2))):
        p = P(win, win, s, False)
        plan = lcnn.pool_tune(n, c, h, h, layout, p)
        assert plan.tuned == 1 and plan.us > 0 and 1 <= plan.fh <= 4 and 1 <= plan.fw <= 4
        again = lcnn.pool_plan_lookup(n, c, h, h, layout, p)
        assert again.as_tuple() == plan.as_tuple() and again.tuned == 1
        x = rng_uniform(h + c, n * c * h * h)
        t = dev(x, (n, c, h, h), layout, cuda)
        want, _ = C.pool_plain(x, n, c, h, h, layout, win, win, s, False)
        got, rep = lcnn.pool_layout(t, p)  # runs the cached plan
        assert bit_equal(got.to_host(), want), (layout, n, c, h, plan)
        got, rep = lcnn.pool_run_plan(t, p, plan)
        assert bit_equal(got.to_host(), want)
        # every explicit plan of the search space, including NCHW ring shapes
        for fh in (1, 2, 3, 4):
            for fw in ((1, 2) if layout == NCHW else (1, 2, 3, 4)):
                q = capi.PoolPlan(fh, fw, 0, 0, 0, 0, 0.0)
                got, _ = lcnn.pool_run_plan(t, p, q)
                assert bit_equal(got.to_host(), want), (layout, fh, fw)
        if layout == NCHW:
            for ring in ((48, 2, 2), (24, 2, 4), (16, 3, 4), (12, 4, 4)):
                q = capi.PoolPlan(plan.fh, plan.fw, *ring, 0, 0.0)
                try:
                    got, _ = lcnn.pool_run_plan(t, p, q)
                except Exception:
                    continue  # a ring too small for this shape's rows is refused
                assert bit_equal(got.to_host(), want), (layout, ring)
