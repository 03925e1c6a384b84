"""`bench.py --impl reference` on the host cores (no GPU): one JSON line with the
engine arm's metric / unit / config vocabulary, `impl`, a `cpu_baseline`
describing the run and a zero-copy `e2e` -- the unmodified reference from
baseline/_ref when it is installed, the oracle port otherwise."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_prints_the_contract_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(rows) == 1
    line = json.loads(rows[0])
    assert line["impl"] == "reference" and line["unit"] == "DOF*steps/s" and line["higher_is_better"] is True
    assert line["metric"].startswith("DOF*steps/s") and line["dtype"] == "f64" and line["value"] > 1e6
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert "ensemble members" in cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    if (ROOT / "baseline" / "_ref" / "curvipat" / "__init__.py").exists():
        assert cb["kind"] == "reference"


def test_reference_arm_is_silent_on_other_ranks():
    import os

    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""
