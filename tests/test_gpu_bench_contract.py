"""bench.py's GPU arm on the box: the JSON line the driver parses (the headline metric,
device value, end-to-end value through the C ABI with host buffers, roofline of the
rollout kernel, clocks, the launch count and the same-run CPU baseline)."""
import importlib.util
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_gpu_arm_json_line():
    spec = importlib.util.spec_from_file_location("bench_contract_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-extras", "--no-c5"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["metric"] == bench.METRIC and line["unit"] == "rollouts/s" and "impl" not in line
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3
    assert line["config"] == json.loads(json.dumps(bench.CONFIG))
    assert line["higher_is_better"] is True and line["vs_baseline"] is None
    B = bench.K_SAMPLES + 1
    assert line["value"] > 0.0
    assert abs(line["ms_per_step"] - 1e3 * B / line["value"]) < 1e-6 * line["ms_per_step"]
    # end to end through the C ABI with host buffers: the noise matrix goes up every step
    e2e = line["e2e"]
    assert e2e["unit"] == "rollouts/s" and 0.0 < e2e["value"] <= 1.05 * line["value"]
    assert e2e["h2d_bytes_per_step"] >= bench.K_SAMPLES * bench.HORIZON * 8 and e2e["d2h_bytes_per_step"] > 0
    # roofline of the rollout kernel: achieved = algorithmic flop per launch / live kernel time
    rf = line["roofline"]
    assert rf["unit"] == "TFLOP/s" and 0.0 < rf["frac"] < 1.0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert abs(rf["achieved"] - rf["flop_per_launch"] / (rf["kernel_ms"] * 1e-3) * 1e-12) < 1e-6 * rf["achieved"]
    assert rf["kernel_ms"] <= line["ms_per_step"]
    clk = line["clocks"]
    assert clk["sm_mhz"] > 0 and isinstance(clk["reasons"], list)
    assert line["gpu_launches"] == 3 * line["steps"]  # rollouts + softmax partial + combine per iteration
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["value"] > 0.0 and cb["unit"] == "rollouts/s"
