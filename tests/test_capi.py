"""CPU-only checks of the drop-in boundary: the sm_100a library loads, exports
every symbol include/lcnn_cuda.h declares, and enforces the reference's
validation rules (layout.cpp:13-26, pool.cpp:19-26/182-191, softmax.cpp) before
touching the device."""
import ctypes
import subprocess

import pytest

from paper_1610_03618_b200 import capi, errors, lcnn

DUMMY = ctypes.c_void_p(256)  # never dereferenced: validation fails first


def test_library_exports_every_declared_symbol():
    lib = capi.lib()
    declared = capi.declared_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = {line.split()[-1] for line in nm.splitlines() if " T " in line}
    assert set(declared) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_basics():
    lib = capi.lib()
    assert lib.lcnn_abi_version() == 1
    assert lib.lcnn_status_name(4) == b"PlanError"
    assert lib.lcnn_flattenable_pair(capi.CHWN, capi.NCHW) == 1
    assert lib.lcnn_flattenable_pair(capi.NCHW, capi.CHWN) == 1
    assert lib.lcnn_flattenable_pair(capi.NCHW, capi.NHWC) == 0
    assert lib.lcnn_flattenable_pair(capi.CHWN, capi.CHWN) == 0


def _st(name, *args):
    return getattr(capi.lib(), name)(*args)


def test_transform_plan_validation(kats):
    t = kats["plan_errors"]["tensor"]
    n, c, h, w = t["dims"]
    for case in kats["plan_errors"]["cases"]:
        st = _st("lcnn_transform_tiled", DUMMY, DUMMY, n, c, h, w, case["src"], case["dst"],
                 case["tile"], int(case["wide"]), None)
        assert st == 4, case["what"]
    with pytest.raises(errors.PlanError, match="wide copy requires N >= 64"):
        capi.check(_st("lcnn_transform_tiled", DUMMY, DUMMY, 32, 3, 5, 5, 1, 0, 32, 1, None))
    with pytest.raises(errors.ShapeError, match="all dims must be >= 1"):
        capi.check(_st("lcnn_transform", DUMMY, DUMMY, 0, 3, 5, 5, 1, 0, None))


def test_pool_validation(kats):
    with pytest.raises(errors.ShapeError, match="window larger than image"):
        capi.check(_st("lcnn_pool_layout", DUMMY, DUMMY, 1, 1, 3, 3, 0, 4, 4, 1, 0, None, None))
    with pytest.raises(errors.ShapeError, match="window and stride must be >= 1"):
        capi.check(_st("lcnn_pool_layout", DUMMY, DUMMY, 1, 1, 3, 3, 0, 2, 2, 0, 0, None, None))
    with pytest.raises(errors.LayoutError, match="only CHWN and NCHW"):
        capi.check(_st("lcnn_pool_layout", DUMMY, DUMMY, 2, 2, 4, 4, capi.NHWC, 2, 2, 2, 0, None,
                       None))
    for case in kats["pool_plan_errors"]["cases"]:
        st = _st("lcnn_pool_coarsened", DUMMY, DUMMY, 2, 2, 8, 8, case["layout"], 2, 2, 2, 0,
                 *case["plan"], None, None)
        assert capi.lib().lcnn_status_name(st).decode() == case["error"]
    ho, wo = lcnn.pool_output_extents(55, 55, lcnn.PoolParams(3, 3, 2))
    assert (ho, wo) == (27, 27)
    assert lcnn.pool_output_extents(224, 224, lcnn.PoolParams(2, 2, 2)) == (112, 112)


def test_softmax_and_conv_validation():
    with pytest.raises(errors.ShapeError, match="softmax: empty matrix"):
        capi.check(_st("lcnn_softmax_fused", DUMMY, DUMMY, 0, 10, 16384, None, None, None))
    assert capi.lib().lcnn_softmax_reference_scratch_bytes(4, 10) == (8 + 80) * 4
    ho, wo = ctypes.c_uint32(), ctypes.c_uint32()
    capi.call("lcnn_conv_output_extents", 227, 227, 11, 11, 4, 0, ctypes.byref(ho),
              ctypes.byref(wo))
    assert (ho.value, wo.value) == (55, 55)
    with pytest.raises(errors.ShapeError):
        capi.call("lcnn_conv_output_extents", 3, 3, 5, 5, 1, 0, ctypes.byref(ho), ctypes.byref(wo))


def test_make_plan_mirror(kats):
    for case in kats["make_plan"]["cases"]:
        p = lcnn.make_plan(case["src"], case["dst"], *case["dims"])
        assert (p.kind == lcnn.TILED_2D) == (case["kind"] == "tiled")
        if case["kind"] == "tiled":
            assert p.tile == case["tile"] and p.wide_copy == case["wide"]


def test_sync_word_entry_points_validate_before_the_device():
    """lcnn_*_forward_packed_ex reject a misaligned sync word (and the plain
    entries' null checks) with LCNN_EINVAL (11) before any device work."""
    lib = capi.lib()
    odd = ctypes.c_void_p(256 + 4)
    st = lib.lcnn_fc_forward_packed_ex(DUMMY, capi.NCHW, DUMMY, DUMMY, 128, 4096, 9216,
                                       capi.PREC_TF32, None, 0, odd, None, 0, None)
    assert st == 11 and b"sync word" in lib.lcnn_last_error()
    st = lib.lcnn_conv_forward_packed_ex(DUMMY, DUMMY, DUMMY, 128, 384, 13, 13, capi.CHWN, 256,
                                         3, 3, 1, 1, capi.PREC_TF32, None, 0, odd, None)
    assert st == 11 and b"sync word" in lib.lcnn_last_error()
    st = lib.lcnn_fc_forward_packed_ex(None, capi.NCHW, DUMMY, DUMMY, 128, 4096, 9216,
                                       capi.PREC_TF32, None, 0, None, None, 0, None)
    assert st == 11 and b"null" in lib.lcnn_last_error()
