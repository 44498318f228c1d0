"""bench.py's output contract: one JSON line with the keys the driver reads
(both arms), checked on a quick CPU run of the reference arm and on a short
GPU run of the product arm."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([sys.executable, str(ROOT / "bench.py")] + args, capture_output=True, text=True,
                         timeout=timeout, env=e, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _check_common(line):
    assert BASE_KEYS <= set(line), sorted(BASE_KEYS - set(line))
    assert line["metric"] == json.loads((ROOT / "BASELINE.json").read_text())["metric"]
    assert line["unit"] == "MLUP/s" and line["higher_is_better"] is True
    assert line["scaling"] == "weak" and line["dtype"] == "f64" and line["vs_baseline"] is None
    assert "workload" in line["config"] and line["config"]["sweeps_per_step"] == 100
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(line["e2e"])


def test_reference_arm_line():
    line = _run(["--impl", "reference", "--steps", "2", "--warmup", "1"],
                env={"SB200_BENCH_CPU_N": "64"}, timeout=300)
    _check_common(line)
    assert line["impl"] == "reference" and line["value"] > 0
    cpu = line["cpu_baseline"]
    assert cpu["kind"] == "port" and cpu["cores"] >= 1 and cpu["variant"] in cpu["variants"]
    assert cpu["value"] == line["value"] == line["e2e"]["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_product_arm_line():
    line = _run(["--steps", "2", "--warmup", "3", "--no-cpu", "--no-also"], timeout=900)
    _check_common(line)
    assert "impl" not in line and line["n_gpus"] == 1 and line["steps"] == 2 and line["warmup"] == 3
    assert line["value"] > 1e5  # > 100 GLUP/s: the CUDA path ran
    assert line["gpu_launches"] == 2 * 25
    roof = line["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(roof)
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s"
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] == e2e["d2h_bytes_per_step"] == 1026 ** 3 * 8
    assert e2e["value"] < line["value"]  # copies inside the timed region
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])
