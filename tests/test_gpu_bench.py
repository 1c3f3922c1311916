"""The bench.py contract on a B200: one JSON line per run with the keys the
driver and the judge read (metric/value/unit, roofline, cpu_baseline, e2e,
clocks, gpu_launches), for a single-op workload and for the whole-network
workload.  The reference arm (CPU only) is covered by test_bench_reference.py."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(*args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    return json.loads(lines[0])


def _check_common(d, steps):
    assert BASE_KEYS <= d.keys(), BASE_KEYS - d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] >= 3
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert "workload" in d["config"]
    rl = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rl, k
    assert rl["achieved"] > 0 and rl["peak"] > 0
    assert abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-3
    e2e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e2e, k
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    assert d["gpu_launches"] > 0


def test_bench_single_op_line():
    d = _run("--workload", "pl5", "--steps", "5", "--warmup", "3", "--ref-sample-gb", "0.05")
    _check_common(d, 5)
    assert d["unit"] == "GB/s" and d["roofline"]["bound"] == "hbm"
    cb = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in cb, k
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] > 0


def test_bench_network_line():
    d = _run("--workload", "alexnet", "--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    _check_common(d, 5)
    assert d["unit"] == "images/s" and d["roofline"]["bound"] == "tensor"
    assert d["roofline"]["per_entry_us"]
