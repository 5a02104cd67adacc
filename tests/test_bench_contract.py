"""bench.py JSON lines against the driver contract: the reference arm on CPU, the product arm on the GPU."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "r8",
                          "--steps", "2", "--warmup", "3", "--cpu-budget", "0.5", "--no-numba"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "GMAC/s" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "GMAC/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert "ResNet-8" in line["config"]["workload"] and line["config"]["batch_per_gpu"] == 1024
    assert line["steps"] == 2 and line["warmup"] == 3
    # the same config dict the product arm prints (the driver compares them)
    sys.path.insert(0, str(ROOT))
    import argparse

    import bench
    from paper_2002_09481_b200 import resnet

    spec = bench.workload_spec("r8", "trunc2")
    want = bench.make_config(spec, argparse.Namespace(), 1024, 1, resnet.macs_per_image(spec["nodes"]))
    assert line["config"] == want


def test_default_workload_is_the_north_star_config():
    """BASELINE configs[2] (ResNet-50 224x224, batch 256) is what a bare `bench.py` measures."""
    sys.path.insert(0, str(ROOT))
    import bench

    src = (ROOT / "bench.py").read_text()
    assert 'ap.add_argument("--workload", default="r50"' in src
    spec = bench.workload_spec("r50", "trunc2")
    assert spec["batch"] == 256 and "ResNet-50" in spec["desc"] and "224x224" in spec["desc"]


@pytest.mark.gpu
def test_b200_arm_json_line():
    """The product arm's line carries every contract key with the right types (a short run)."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3",
                          "--cpu-budget", "0.5"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["unit"] == "GMAC/s" and line["value"] > 0 and line["n_gpus"] == 1 and line["steps"] == 3
    assert isinstance(line["gpu_launches"], int) and line["gpu_launches"] > 0
    roof = line["roofline"]
    assert 0 < roof["frac"] <= 1 and roof["achieved"] > 0 and roof["peak"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    assert line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["cpu_baseline"]["value"] > 0 and line["cpu_baseline"]["cores"] >= 1
    assert set(line["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert line["parity"]["status"] == "bit-exact", line["parity"]
    assert line["config"]["batch_per_gpu"] == 256 and "ResNet-50" in line["config"]["workload"]
    hbm = line["hbm"]
    assert {"quantize", "pool"} <= set(hbm["kernels"]) and all(v["gbs"] > 0 for v in hbm["kernels"].values())
    assert line["roofline"]["dominant_kernel"] in line["roofline"]["kernels"]
