"""bench.py's JSON line (the driver's contract): one line with the required keys,
the roofline and cpu_baseline objects, e2e with the bytes copied per step, clocks
sampled during the timed region; and the reference arm's line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_has_the_contract_keys():
    d = _run(["--steps", "4", "--warmup", "3", "--no-sweep", "--no-extra", "--cpu-tokens", "16"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] >= 3 and d["value"] > 0
    assert d["config"]["workload"] == "mixtral_prefill" and d["dtype"] == "bf16"
    ro = d["roofline"]
    assert ro["bound"] in ("tensor", "hbm") and ro["unit"] in ("TFLOP/s", "GB/s")
    assert 0 < ro["achieved"] and 0 < ro["peak"] and abs(ro["frac"] - ro["achieved"] / ro["peak"]) < 1e-9
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == d["steps"] * len([k for k in d["kernel_ms"] if not k.startswith("_")])
    assert d["kernel_ms"]["_events_tile_step"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-tokens", "8"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["dtype"] == "f64"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
