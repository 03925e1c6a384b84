"""bench.py's one-line JSON contract on a real GPU (a short run: 1 bench step of
5 time steps, no extras): every key the driver reads is present and
consistent -- metric / value / unit, e2e through the public API with its byte
counts, the roofline object of the dominant kernel, kernels launched, clocks."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "1", "--warmup", "3", "--chunk", "5",
                        "--no-extras"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(rows) == 1, r.stdout[-2000:]
    return json.loads(rows[0])


def test_headline_keys(line):
    assert line["metric"].startswith("DOF*steps/s") and line["unit"] == "DOF*steps/s"
    assert line["n_gpus"] == 1 and line["steps"] == 1 and line["warmup"] == 3
    assert line["higher_is_better"] is True and line["dtype"] == "f64" and line["vs_baseline"] is None
    assert line["scaling"] in ("weak", "strong") and "synthetic" in line["data"]
    assert "workload" in line["config"] and "model" not in line["config"]
    dof = line["config"]["dof"]
    assert line["value"] == pytest.approx(dof * 5 / (line["ms_per_step"] / 1e3), rel=1e-6)
    assert line["value"] > 1e9 and line["finite"] is True and line["diverged_runs"] == 0


def test_e2e_goes_through_host_buffers(line):
    e = line["e2e"]
    assert e["unit"] == line["unit"] and 0 < e["value"] <= line["value"] * 1.05
    assert e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 512 * 2 * 128 * 256 * 8
    assert e["value"] != line["value"]


def test_roofline_object(line):
    rf = line["roofline"]
    assert rf["bound"] in ("tensor", "hbm") and rf["unit"] in ("TFLOP/s", "GB/s")
    assert rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"], rel=1e-9) and 0 < rf["frac"] < 1
    assert rf["traffic"] is None or rf["traffic"] > 0
    names = [k["kernel"] for k in line["kernels"]]
    assert rf["kernel"] in names
    assert sum(k["share_of_step"] for k in line["kernels"]) == pytest.approx(1.0, abs=1e-6)


def test_launch_count_and_clocks(line):
    # two kernels per time step and lane (fused front + rho GEMM), two lanes, 5 time steps, + the step-counter set per lane
    assert line["gpu_launches"] >= 2 * 2 * 5
    cl = line["clocks"]
    assert 500 < cl["sm_mhz"] <= cl["sm_max_mhz"] and isinstance(cl["reasons"], list)
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(cl["reasons"])
