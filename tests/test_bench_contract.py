"""bench.py's JSON-line contract (the driver parses it): both arms print ONE line with
the keys the task's bench contract and ④ name.  The reference arm (the float64 oracle
on the host cores) runs here on CPU; the kk arm needs the GPU."""
import json
import os
import subprocess
import sys

import pytest

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(root, *args, timeout):
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], cwd=root, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line(root):
    d = run_bench(root, "--impl", "reference", "--steps", "1", "--warmup", "3", "--ref-workers", "2", "--pool", "4",
                  timeout=600)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["steps"] == 1 and d["warmup"] >= 3 and d["n_gpus"] == 1
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and d["vs_baseline"] is None
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert cb["cpu_model"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_kk_arm_line(root):
    d = run_bench(root, "--steps", "3", "--warmup", "3", "--batch", "16", "--pool", "16", "--no-cpu-baseline",
                  "--no-cufft", timeout=900)
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["dtype"] == "f32" and d["scaling"] == "weak" and d["vs_baseline"] is None
    assert d["config"]["workload"].startswith("C5")
    rf = d["roofline"]
    assert rf["bound"] in ("alu", "hbm", "tensor") and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    # the end-to-end leg cannot beat the copies it contains (5 % timing slack)
    assert e["value"] <= 1.05 * e["pcie_ceiling"]["value"]
    assert e["value"] < d["value"]
    assert d["errors"]["bits"] > 0
    # weak scaling over the sharded 4096-buffer stream: 3 steps x 16 buffers, counted from the counters
    assert d["config"]["buffers_timed"] == 3 * 16 and d["config"]["stream_buffers"] == 4096
    assert d["comm"]["world"] == 1
