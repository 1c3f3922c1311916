"""The `lcnn` command-line tool (tools/lcnn.cpp): the reference CLI's
subcommands, options, CSV outputs and exit codes (reference
tools/lcnn.cpp:58-246).  CPU tests cover parsing, usage errors and the
fixture table (checked against the reference library's fixture_list_csv);
the GPU test runs `run-net` and compares every column of the timing CSV
except the time itself with the reference CLI body run on the same network
and seed (oracle/ref_shim.cpp ref_run_net_cli)."""
import csv
import io
import os
import subprocess

import pytest

from oracle.oracle import REF_LIB, Ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "build", "tools", "lcnn")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="build/tools/lcnn not built")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


_REF_SNIPPET = """
import ctypes, sys
lib = ctypes.CDLL(sys.argv[1])
fn = getattr(lib, sys.argv[2])
fn.restype = ctypes.c_char_p
if sys.argv[2] == "ref_fixture_list_csv":
    fn.argtypes = [ctypes.c_uint32]
    r = fn(int(sys.argv[3]))
else:
    fn.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64]
    r = fn(open(sys.argv[3], "rb").read(), sys.argv[4].encode(), int(sys.argv[5]))
if r is None:
    sys.exit(lib.ref_last_error and 3)
sys.stdout.write(r.decode())
"""


def ref_call(fn, *args):
    """A reference-library string entry point, called in a fresh interpreter:
    the unmodified reference builds its CSV text with libstdc++ streams,
    which must not share a process with the venv's numpy runtime libraries
    (observed to crash inside the reference's ostringstream)."""
    if not Ref.available():
        pytest.skip("reference library (oracle/_ref) not built")
    import sys

    r = subprocess.run([sys.executable, "-c", _REF_SNIPPET, REF_LIB, fn, *map(str, args)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return r.stdout


def test_help_and_usage_errors():
    r = run("--help")
    assert r.returncode == 0 and "run-net" in r.stdout and "bench-transform" in r.stdout
    assert run().returncode == 1                        # a subcommand is required
    r = run("bogus")
    assert r.returncode == 1 and "unknown subcommand" in r.stderr
    assert run("run-net").returncode == 1               # CONFIG is required
    assert run("fixtures").returncode == 1              # nothing to do (try --list)
    assert run("fixtures", "--scale", "x", "--list").returncode == 1
    assert run("bench-layer", "--nope").returncode == 1
    r = run("bench-transform", "--dims", "64x96")
    assert r.returncode == 1 and "--dims must look like" in r.stderr
    r = run("bench-layer", "--id", "NOPE")
    assert r.returncode == 1 and "unknown fixture id" in r.stderr
    r = run("run-net", os.path.join(ROOT, "configs", "mininet.json"), "--preset", "titan-z")
    assert r.returncode == 1 and "unknown preset" in r.stderr


@pytest.mark.parametrize("scale", [1, 4])
def test_fixtures_list_matches_reference(scale, tmp_path):
    want = ref_call("ref_fixture_list_csv", scale)
    r = run("fixtures", "--list", "--scale", str(scale))
    assert r.returncode == 0 and r.stdout == want
    out = tmp_path / "fx.csv"                           # --out before the subcommand
    assert run("--out", str(out), "fixtures", f"--scale={scale}", "--list").returncode == 0
    assert out.read_text() == want


@pytest.mark.gpu
@pytest.mark.parametrize("preset", ["titan-black", "titan-x"])
def test_run_net_matches_reference_cli(preset, tmp_path):
    cfg = os.path.join(ROOT, "configs", "mininet.json")
    want = ref_call("ref_run_net_cli", cfg, preset, 7)
    out = tmp_path / "run.csv"
    r = run("run-net", cfg, "--preset", preset, "--seed", "7", "--out", str(out))
    assert r.returncode == 0, r.stderr
    got = list(csv.DictReader(io.StringIO(out.read_text())))
    ref = list(csv.DictReader(io.StringIO(want)))
    assert [k for k in got[0]] == [k for k in ref[0]]
    for g, w in zip(got, ref):
        for key in g:
            if key != "nanos":
                assert g[key] == w[key], (key, g, w)
        assert int(g["nanos"]) > 0
    assert len(got) == len(ref)


@pytest.mark.gpu
def test_bench_transform_and_layer_rows():
    r = run("bench-transform", "--dims", "64x8x13x13", "--repeats", "2")
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert rows and all(float(x["gbps"]) > 0 for x in rows if "gbps" in x)
    r = run("bench-layer", "--id", "PL5", "--scale", "8", "--repeats", "2")
    assert r.returncode == 0, r.stderr
    assert len(list(csv.DictReader(io.StringIO(r.stdout)))) >= 2
