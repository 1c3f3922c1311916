"""The reference's OWN unit tests (/root/reference/proj/tests/test_*.cpp) and
its acceptance gate, compiled unchanged against the B200 lcnn library by
tests/cpp/build_ref_tests.sh (binaries in build/reftests/, built in the
container that has /root/reference and shipped with the snapshot).  This is
the drop-in proof: the reference's API, error types and tolerances hold with
every hot op running on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "reftests")
SUITES = ["test_tensor", "test_layout", "test_pool", "test_softmax", "test_select", "test_conv",
          "test_net", "test_bench"]


def _run(name, timeout=900):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    return subprocess.run([path], capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def test_reference_tensor_suite_cpu():
    """test_tensor.cpp touches no kernel: it runs here too."""
    r = _run("test_tensor")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite(cuda, suite):
    r = _run(suite)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_reference_acceptance_gate(cuda):
    r = _run("acceptance", timeout=1200)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "all criteria passed" in r.stdout
