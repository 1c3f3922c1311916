"""GPU parity: the fused softmax kernel and the five-kernel baseline against
the CPU oracle (which is bit-identical to the reference, same libm expf).
Tolerance: approx_equal 1e-6 (tensor.cpp:157-187, bench.cpp:158/169) -- the
GPU's parallel reduction order and CUDA expf (<= 2 ulp) are the only
differences."""
import math

import numpy as np
import pytest

from oracle.oracle import C, approx_equal, rng_uniform
from paper_1610_03618_b200 import errors, lcnn

pytestmark = pytest.mark.gpu
TOL = 1e-6


def dev(x, r, c, device):
    return lcnn.DeviceMatrix.from_host(x, r, c, device=device)


def test_kats(cuda, kats):
    k = kats["softmax_closed_forms"]
    for fn in (lambda m: lcnn.softmax_fused(m)[0], lambda m: lcnn.softmax_reference(m)[0]):
        out = fn(dev(np.zeros(30, np.float32), 3, 10, cuda)).to_host()
        assert np.allclose(out, 0.1, rtol=TOL, atol=0)
        out = fn(dev(np.array(k["ln2"]["input"], np.float32), 1, 2, cuda)).to_host()
        assert np.allclose(out, k["ln2"]["expected"], rtol=TOL, atol=0)
        out = fn(dev(np.array([1000.0, 1000.0], np.float32), 1, 2, cuda)).to_host()
        assert np.allclose(out, 0.5, rtol=TOL, atol=0)
        out = fn(dev(np.array([-44.0, 0.0, 17.5], np.float32), 3, 1, cuda)).to_host()
        assert out.tolist() == [1.0, 1.0, 1.0]
    p = kats["softmax_pass_accounting"]
    m = dev(rng_uniform(5, 160, -5, 5), 16, 10, cuda)
    rep = lcnn.softmax_reference(m)[1]
    assert (rep.materializations, rep.full_matrix_sweeps) == (3, 8)
    rep = lcnn.softmax_fused(m)[1]
    assert (rep.materializations, rep.full_matrix_sweeps) == (0, 2)
    s = p["streaming"]
    x = rng_uniform(6, s["rows"] * s["cols"], -5, 5)
    got, rep = lcnn.softmax_fused(dev(x, s["rows"], s["cols"], cuda), local_buffer_limit=s["limit"])
    assert rep.full_matrix_sweeps == 5
    assert approx_equal(got.to_host(), C.softmax_reference(x, s["rows"], s["cols"])[0], TOL)


def test_nonfinite_raises_domain_error(cuda):
    for v in (math.inf, -math.inf, math.nan):
        for cols in (3, 1000, 5000, 20000):
            x = np.zeros(2 * cols, np.float32)
            x[-1] = v
            m = dev(x, 2, cols, cuda)
            with pytest.raises(errors.DomainError):
                lcnn.softmax_fused(m)
            with pytest.raises(errors.DomainError):
                lcnn.softmax_reference(m)
    # the flag is reset per call: a clean call after a bad one passes
    lcnn.softmax_fused(dev(np.zeros(6, np.float32), 2, 3, cuda))


def test_reference_fixtures(cuda, ref_vectors):
    v = ref_vectors
    keys = sorted({k.split("_")[1] for k in v.files if k.startswith("softmax_")}, key=int)
    for k in keys:
        r, c = v[f"softmax_{k}_meta"].tolist()
        m = dev(v[f"softmax_{k}_in"], r, c, cuda)
        assert approx_equal(lcnn.softmax_fused(m)[0].to_host(), v[f"softmax_{k}_fused"], TOL), k
        assert approx_equal(lcnn.softmax_reference(m)[0].to_host(), v[f"softmax_{k}_ref"], TOL), k


@pytest.mark.parametrize("cols", [1, 3, 10, 16, 17, 63, 64, 100, 256, 257, 512, 999, 1000, 1024,
                                  1025, 2048, 2049, 4096, 4097, 8192, 10000, 12288, 16384, 16385,
                                  16388, 28000, 40000, 56000, 60000])
def test_every_kernel_shape(cuda, cols):
    for rows in (1, 7, 33):
        x = rng_uniform(rows * cols, rows * cols, -5, 5)
        m = dev(x, rows, cols, cuda)
        want, _ = C.softmax_fused(x, rows, cols)
        got = lcnn.softmax_fused(m)[0].to_host()
        assert approx_equal(got, want, TOL), (rows, cols)
        sums = got.reshape(rows, cols).astype(np.float64).sum(axis=1)
        assert np.all(np.abs(sums - 1.0) <= 1e-5)
        got5 = lcnn.softmax_reference(m)[0].to_host()
        assert approx_equal(got5, want, TOL)


def test_config2_batches(cuda):
    """Config 2: N in {128..4096} x 1000 classes, fused and five-pass."""
    for rows in (128, 256, 512, 1024, 2048, 4096):
        x = rng_uniform(rows, rows * 1000, -5, 5)
        want, _ = C.softmax_fused(x, rows, 1000)
        m = dev(x, rows, 1000, cuda)
        assert approx_equal(lcnn.softmax_fused(m)[0].to_host(), want, TOL)
        assert approx_equal(lcnn.softmax_reference(m)[0].to_host(), want, TOL)


def test_shift_invariance_and_monotone(cuda):
    x = rng_uniform(7, 5 * 40, -5, 5)
    base = lcnn.softmax_fused(dev(x, 5, 40, cuda))[0].to_host()
    for c in (-50.0, -1.5, 13.0, 50.0):
        got = lcnn.softmax_fused(dev(x + np.float32(c), 5, 40, cuda))[0].to_host()
        assert approx_equal(got, base, TOL)
    x = rng_uniform(8, 6 * 12, -5, 5).reshape(6, 12)
    out = lcnn.softmax_fused(dev(x, 6, 12, cuda))[0].to_host().reshape(6, 12)
    for i in range(6):
        order = np.argsort(x[i])
        assert np.all(np.diff(out[i][order]) > 0)


@pytest.mark.parametrize("rows,cols", [(300, 20000), (457, 16388), (200, 40000)])
def test_wide_rows_persistent_smem_kernel(cuda, rows, cols):
    """Rows beyond the register kernels are staged in shared memory by
    persistent CTAs (double-buffered bulk copies when two rows fit): more
    rows than CTAs, so every buffer is refilled several times; within 1e-6 of
    the oracle, and a non-finite entry still sets the flag."""
    x = rng_uniform(rows + cols, rows * cols, -5, 5)
    m = dev(x, rows, cols, cuda)
    want, _ = C.softmax_fused(x, rows, cols)
    got = lcnn.softmax_fused(m)[0].to_host()
    assert approx_equal(got, want, TOL), (rows, cols)
    x2 = x.copy()
    x2[(rows - 1) * cols + 5] = np.inf
    with pytest.raises(errors.DomainError):
        lcnn.softmax_fused(dev(x2, rows, cols, cuda))
