"""bench.py's reference arm (the CPU path of the headline metric, runnable without a GPU)
prints the one-line JSON contract the driver parses: metric / unit / config shared with
the GPU arm, `impl: reference`, a `cpu_baseline` describing the run, and an `e2e` object
repeating the line's own value with zero transfer bytes."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def _run(extra_env=None):
    env = {**os.environ, **(extra_env or {})}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                         text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()


def test_reference_arm_line():
    lines = _run()
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "SH transform pairs/s (fp64)" and d["unit"] == "field-pairs/s"
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and d["vs_baseline"] is None
    assert d["config"]["workload"].startswith("config1:") and d["config"]["fields"] == 15
    assert d["config"]["R"] == 255 and d["config"]["grid"] == [768, 384]
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["steps"] == 1 and d["warmup"] >= 3
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_only_rank_zero_prints():
    """Under torchrun (N > 1) rank 0 alone runs and prints the reference line."""
    assert _run({"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"}) == []


@pytest.mark.gpu
def test_gpu_arm_line():
    """The GPU arm's line on a short run: the headline config, a roofline object for the
    dominant kernel measured live, an end-to-end number with its transfer bytes, the
    library's own launch count and the clocks sampled during the timed region."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3",
                          "--warmup", "3", "--soak", "0", "--no-cpu-baseline", "--no-mlsdc"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["metric"] == "SH transform pairs/s (fp64)" and d["unit"] == "field-pairs/s"
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["dtype"] == "f64" and d["scaling"] == "weak"
    assert d["config"]["workload"].startswith("config1:") and d["vs_baseline"] is None
    assert d["value"] > 1e4 and d["gpu_launches"] >= 4 * 3
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert 0.0 < r["frac"] < 1.0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    tri = 15 * 256 * 257 // 2 * 16
    assert e["h2d_bytes_per_step"] == tri and e["d2h_bytes_per_step"] == tri
    assert 0 < e["value"] < d["value"] and e["roundtrip_err"] < 1e-12
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] >= c["sm_mhz"] and isinstance(c["reasons"], list)
    assert d["roundtrip_err"] < 1e-12
