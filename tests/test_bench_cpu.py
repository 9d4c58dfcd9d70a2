"""CPU: bench.py's contract pieces that do not need a GPU -- the reference arm
(oracle port on host cores) end to end, the CPU-baseline record, and the
roofline / path-roofline arithmetic."""

import json
import subprocess
import sys
from pathlib import Path
from types import SimpleNamespace

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def _args(**kw):
    base = dict(gpus=1, steps=2, warmup=1, impl="reference", streams=64, height=90, width=160,
                drop=0.10, e2e_streams=8, no_e2e=True, no_cpu_baseline=False, cpu_workers=2,
                roofline_steps=3, lanes=2)
    base.update(kw)
    return SimpleNamespace(**base)


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1", "--cpu-workers", "2",
                          "--height", "90", "--width", "160"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] == 2
    assert line["metric"] == bench.METRIC and "workload" in line["config"]


def test_cpu_baseline_record():
    rec = bench.cpu_baseline(_args())
    assert rec["unit"] == "frames/s" and rec["value"] > 0 and rec["cores"] == 2
    assert "oracle" in rec["sample"]


def test_roofline_arithmetic():
    a = _args(height=1080, width=1920, steps=20)
    stages = {"K1_encode": (1.0 * 6, 6), "K5_upscale_blend": (1.25 * 6, 6)}
    r = bench.roofline(a, stages, 32)
    assert r["kernel"] == "K5_upscale_blend" and r["bound"] == "hbm" and r["unit"] == "GB/s"
    frame = 1080 * 1920 * 3 * 4
    assert r["algorithmic_bytes_per_launch"] > 32 * 9 * frame
    assert r["achieved"] == pytest.approx(r["algorithmic_bytes_per_launch"] / 1.25e-3 / 1e9, rel=1e-3)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)
    p = bench.path_roofline(a, 100000.0)
    assert p["bytes_per_frame"] == 1080 * 1920 * 3 * 8
    assert p["roofline_fps"] == pytest.approx(p["peak"] * 1e9 / p["bytes_per_frame"], rel=1e-6)


def test_scale_schedule_half_and_half():
    for k in range(8):
        assert {bench.scale_of(0, k), bench.scale_of(1, k)} == {2, 3}
