"""bench.py's reference arm on the host (the driver runs it beside the GPU arm): one
full C4 MPPI iteration on the reference's own compiled core (oracle/_ref; the C port
when that is not built), and the JSON line the driver parses -- same metric, unit and
config dict as the GPU arm, impl "reference", cpu_baseline and e2e describing the
same run.  Also the torchrun convention: ranks other than 0 exit 0 without work."""
import importlib.util
import json
import os
import subprocess
import sys

from conftest import ROOT


def _bench_module():
    spec = importlib.util.spec_from_file_location("bench_contract_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=e,
                          capture_output=True, text=True, timeout=900)


def test_reference_arm_json_line():
    bench = _bench_module()
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRIC and line["unit"] == "rollouts/s"
    assert line["higher_is_better"] is True and line["n_gpus"] == 1 and line["steps"] == 1
    assert line["config"] == json.loads(json.dumps(bench.CONFIG))  # the GPU arm prints the same dict
    assert line["value"] > 0.0
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["value"] == line["value"] and cb["cores"] >= 1
    assert cb["unit"] == "rollouts/s" and "4097" in cb["sample"]  # full iterations, no extrapolation
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["unit"] == line["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0
    assert abs(line["ms_per_step"] - 1e3 * (bench.K_SAMPLES + 1) / line["value"]) < 1e-6 * line["ms_per_step"]


def test_reference_arm_other_ranks_exit_without_work():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], env={"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""
