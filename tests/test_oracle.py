"""The CPU oracle pinned to the reference: golden KATs from the reference's
own tests, the committed fixtures generated from the reference binary, and
(when oracle/_ref is present) the live reference on fresh seeded inputs."""
import math

import numpy as np
import pytest

from oracle.oracle import CHWN, HWCN, NCHW, NHWC, C, OracleError, Ref, approx_equal, bit_equal, \
    rng_uniform

needs_ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built here")


def test_transform_iota_kat(kats):
    k = kats["transform_iota"]
    x = np.arange(16, dtype=np.float32)
    out = C.transform(x, *k["dims"], k["src_layout"], k["dst_layout"])
    assert out.tolist() == k["expected"]
    back = C.transform(out, *k["dims"], k["dst_layout"], k["src_layout"])
    assert bit_equal(back, x)


def test_pool_kats(kats):
    k = kats["pool_line_average"]
    x = np.arange(1, 13, dtype=np.float32)
    out = C.pool_oracle(x, *k["dims"], NCHW, 1, 4, 2, True)
    assert out.tolist() == k["expected"]
    k = kats["pool_ramp_max"]
    x = np.arange(1, 17, dtype=np.float32)
    assert C.pool_oracle(x, 1, 1, 4, 4, NCHW, 2, 2, 2, False).tolist() == k["expected"]
    with pytest.raises(OracleError):
        C.pool_oracle(np.zeros(9, np.float32), 1, 1, 3, 3, NCHW, 4, 4, 1, False)
    k = kats["pool_line_accounting"]
    x = np.arange(1, 13, dtype=np.float32)
    for layout in (NCHW, CHWN):
        _, rep = C.pool_plain(x, 1, 1, 1, 12, layout, 1, 4, 2, True)
        assert rep == (k["input_loads"], k["output_stores"], k["distinct_inputs"])


def test_coarsened_kats(kats):
    k = kats["pool_coarsened_loads"]
    x = rng_uniform(8, 33, -10, 10)
    out, rep = C.pool_coarsened(x, 1, 1, 3, 11, CHWN, 3, 3, 2, False, 1, 2)
    assert out.size == k["w_out"]
    assert rep[0] == k["coarsened_loads"]
    _, plain = C.pool_plain(x, 1, 1, 3, 11, CHWN, 3, 3, 2, False)
    assert plain[0] == k["plain_loads"]
    assert rep[2] == plain[2]
    for case in kats["pool_plan_errors"]["cases"]:
        with pytest.raises(OracleError) as e:
            C.pool_coarsened(np.zeros(256, np.float32), 2, 2, 8, 8, case["layout"], 2, 2, 2, False,
                             *case["plan"])
        assert e.value.status == {"PlanError": 4, "LayoutError": 3}[case["error"]]


def _model(name):
    if name == "unimodal44":
        return lambda fh, fw: (fh - 4.0) ** 2 + (fw - 4.0) ** 2
    if name == "flat":
        return lambda fh, fw: 1.0
    if name == "inverse_area":
        return lambda fh, fw: 1.0 / (fh * fw)
    return lambda fh, fw: 0.5 if fh == 3 else 1.0


def test_autotune_kats(kats):
    for case in kats["autotune_models"]["cases"]:
        fh, fw = C.autotune(_model(case["model"]))
        assert fh * fw <= 64
        if "expected" in case:
            assert [fh, fw] == case["expected"]
        else:
            assert fh == case["expected_fh"]


def test_softmax_kats(kats):
    k = kats["softmax_closed_forms"]
    tol = k["tolerance"]
    out, _ = C.softmax_reference(np.zeros(30, np.float32), 3, 10)
    assert np.allclose(out, 0.1, rtol=tol, atol=0)
    for fn in (C.softmax_reference, C.softmax_fused):
        out, _ = fn(np.array(k["ln2"]["input"], np.float32), 1, 2)
        assert np.allclose(out, k["ln2"]["expected"], rtol=tol, atol=0)
        out, _ = fn(np.array(k["large_equal"]["input"], np.float32), 1, 2)
        assert np.allclose(out, 0.5, rtol=tol, atol=0)
        out, _ = fn(np.array(k["single_category"]["input"], np.float32), 3, 1)
        assert out.tolist() == [1.0, 1.0, 1.0]
    p = kats["softmax_pass_accounting"]
    x = rng_uniform(5, 160, -5, 5)
    assert C.softmax_reference(x, 16, 10)[1] == (p["reference"]["materializations"],
                                                 p["reference"]["sweeps"])
    assert C.softmax_fused(x, 16, 10)[1] == (0, p["fused"]["sweeps"])
    s = p["streaming"]
    x = rng_uniform(6, s["rows"] * s["cols"], -5, 5)
    got, rep = C.softmax_fused(x, s["rows"], s["cols"], s["limit"])
    assert rep == (0, s["sweeps"])
    assert approx_equal(got, C.softmax_reference(x, s["rows"], s["cols"])[0], 1e-6)
    bad = np.zeros(6, np.float32)
    for v in (math.inf, math.nan):
        bad[5] = v
        with pytest.raises(OracleError) as e:
            C.softmax_fused(bad, 2, 3)
        assert e.value.status == 6
        with pytest.raises(OracleError):
            C.softmax_reference(bad, 2, 3)


def test_select_kats(kats):
    for kind, n, c, ct, nt, want in kats["choose_layout"]["cases"]:
        assert C.choose_layout(kind, n, c, ct, nt) == want
    for fx, (n, c, want) in kats["preference_table"]["fixtures"].items():
        assert C.choose_layout(0, n, c, 32, 128) == want, fx

    def synthetic(layout, n, c):  # test_select.cpp:56-62
        if layout == CHWN:
            return 1.0 if n >= 128 else 3.0
        return 2.0 if c >= 32 else 4.0

    assert list(C.calibrate(synthetic)) == kats["calibration"]["synthetic_crossover"]["expected"]
    assert list(C.calibrate(lambda l, n, c: 1.0 if l == CHWN else 2.0)) == \
        kats["calibration"]["chwn_always_wins"]["expected"]


def test_plan_transforms_kats(kats):
    k = kats["plan_transforms"]
    steps = C.plan_transforms(k["alexnet_chain"]["kinds"], k["alexnet_chain"]["layouts"])
    assert [s[0] for s in steps] == k["alexnet_chain"]["expected_positions"]
    steps = C.plan_transforms(k["lenet_mismatched"]["kinds"], k["lenet_mismatched"]["layouts"])
    assert [list(s) for s in steps] == k["lenet_mismatched"]["expected"]
    assert C.plan_transforms(k["uniform"]["kinds"], k["uniform"]["layouts"]) == []


# ---- pinned to the reference's outputs (committed fixtures) -----------------
def _cases(v, prefix):
    return sorted({key.split("_")[1] for key in v.files if key.startswith(prefix + "_")}, key=int)


def test_oracle_matches_reference_fixtures_transform(ref_vectors):
    v = ref_vectors
    for k in _cases(v, "transform"):
        n, c, h, w, sl, dl = v[f"transform_{k}_meta"].tolist()
        assert bit_equal(C.transform(v[f"transform_{k}_in"], n, c, h, w, sl, dl),
                         v[f"transform_{k}_out"]), k


def test_oracle_matches_reference_fixtures_pool(ref_vectors):
    v = ref_vectors
    for k in _cases(v, "pool"):
        n, c, h, w, layout, wh, ww, s, avg = v[f"pool_{k}_meta"].tolist()
        x = v[f"pool_{k}_in"]
        out, rep = C.pool_plain(x, n, c, h, w, layout, wh, ww, s, avg)
        assert bit_equal(out, v[f"pool_{k}_out"]), k
        assert rep == tuple(v[f"pool_{k}_report"].tolist())
        assert bit_equal(C.pool_oracle(x, n, c, h, w, layout, wh, ww, s, avg), v[f"pool_{k}_oracle"])
        if layout == CHWN:
            for fh, fw in ((2, 2), (1, 3), (3, 1), (4, 4)):
                o2, r2 = C.pool_coarsened(x, n, c, h, w, layout, wh, ww, s, avg, fh, fw)
                assert bit_equal(o2, v[f"pool_{k}_coarse_{fh}x{fw}_out"])
                assert r2 == tuple(v[f"pool_{k}_coarse_{fh}x{fw}_report"].tolist())


def test_oracle_matches_reference_fixtures_softmax(ref_vectors):
    v = ref_vectors
    for k in _cases(v, "softmax"):
        r, c = v[f"softmax_{k}_meta"].tolist()
        x = v[f"softmax_{k}_in"]
        # same libm expf and operation order: bit-identical to the reference
        assert bit_equal(C.softmax_reference(x, r, c)[0], v[f"softmax_{k}_ref"]), k
        assert bit_equal(C.softmax_fused(x, r, c)[0], v[f"softmax_{k}_fused"]), k


def test_oracle_matches_reference_fixtures_conv(ref_vectors):
    v = ref_vectors
    for k in _cases(v, "conv"):
        n, ci, h, w, co, f, stride, pad = v[f"conv_{k}_meta"].tolist()
        out = C.conv_oracle(v[f"conv_{k}_in"], v[f"conv_{k}_filt"], n, ci, h, w, NCHW, co, f, f,
                            stride, pad)
        assert bit_equal(out, v[f"conv_{k}_oracle"]), k


# ---- live reference, fresh inputs --------------------------------------------
@needs_ref
def test_oracle_vs_live_reference_random():
    rng = np.random.default_rng(123)
    for trial in range(40):
        n, c, h, w = (int(x) for x in rng.integers(1, 17, 4))
        sl, dl = [(CHWN, NCHW), (NCHW, CHWN), (NHWC, HWCN), (NCHW, NHWC)][trial % 4]
        x = rng_uniform(trial, n * c * h * w, -100, 100)
        assert bit_equal(C.transform(x, n, c, h, w, sl, dl), Ref.transform(x, n, c, h, w, sl, dl))
    for trial in range(30):  # test_pool.cpp:109-128 shape recipe
        h = int(rng.integers(4, 17))
        win, stride, avg = 2 + trial % 2, 1 + trial % 3, trial % 2
        n, c = (int(x) for x in rng.integers(4, 17, 2))
        x = rng_uniform(100 + trial, n * c * h * h, -10, 10)
        for layout in (NCHW, CHWN):
            a, ra = C.pool_plain(x, n, c, h, h, layout, win, win, stride, avg)
            b, rb = Ref.pool_layout(x, n, c, h, h, layout, win, win, stride, avg)
            assert bit_equal(a, b) and ra == rb
        a, ra = C.pool_coarsened(x, n, c, h, h, CHWN, win, win, stride, avg, 2, 3)
        b, rb = Ref.pool_coarsened(x, n, c, h, h, CHWN, win, win, stride, avg, 2, 3)
        assert bit_equal(a, b) and ra == rb
    for r, c in ((1, 1), (3, 7), (16, 10), (8, 1000), (33, 257)):
        x = rng_uniform(r * c, r * c, -5, 5)
        assert bit_equal(C.softmax_fused(x, r, c)[0], Ref.softmax_fused(x, r, c)[0])
        assert bit_equal(C.softmax_reference(x, r, c)[0], Ref.softmax_reference(x, r, c)[0])


@needs_ref
def test_selector_vs_live_reference(kats):
    rng = np.random.default_rng(7)
    for _ in range(200):
        kind = int(rng.integers(0, 5))
        n, c = int(rng.integers(1, 300)), int(rng.integers(1, 600))
        ct, nt = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        assert C.choose_layout(kind, n, c, ct, nt) == Ref.choose_layout(kind, n, c, ct, nt)
    for case in kats["autotune_models"]["cases"]:
        m = _model(case["model"])
        assert C.autotune(m) == Ref.autotune(m)
