"""bench.py keeps the driver's JSON-line contract: the GPU arm (small C1 run) and the reference arm
(the CPU oracle, no GPU needed) each print one line with the required keys."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout, env=dict(os.environ, RANK="0", WORLD_SIZE="1"))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1"], 600)
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "queries/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C1")


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--config", "C1", "--steps", "3", "--warmup", "3", "--cpu-seconds", "2"], 900)
    assert BASE_KEYS <= d.keys() and "impl" not in d
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "weak" and d["n_gpus"] == 1
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys()
    assert r["bound"] == "hbm" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["gpu_launches"] >= d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert "random_access_roofline" in d
