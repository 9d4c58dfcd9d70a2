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
                roofline_steps=3, lanes=2, scaling="weak")
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
    assert line["cpu_baseline"]["kind"] == bench.reference_kind()
    assert line["cpu_baseline"]["cores"] == 2 and "nproc" in line["cpu_baseline"]["host"]
    assert line["metric"] == bench.METRIC and "workload" in line["config"]
    # same config object as our arm's line, so the driver can pair the two
    assert line["config"] == bench.workload_config(_args(height=90, width=160, steps=2,
                                                         warmup=1))


def test_cpu_baseline_record():
    rec = bench.cpu_baseline(_args())
    assert rec["unit"] == "frames/s" and rec["value"] > 0 and rec["cores"] == 2
    want = "baseline/_ref" if bench.reference_kind() == "reference" else "oracle"
    assert want in rec["sample"]


def test_cpu_arm_port_and_reference_agree(tmp_path):
    # the port (oracle) and, when installed, the unmodified reference give the
    # same reconstruction quality on the same GoP
    if bench.reference_kind() != "reference":
        pytest.skip("baseline/_ref not installed")
    bench._init_worker()
    bench._PREV_OUT.clear()
    _, p_ref = bench._ref_gop(90, 160, 1, 0, 3, 0.1)
    bench._PREV_OUT.clear()
    _, p_port = bench._port_gop(90, 160, 1, 0, 3, 0.1)
    assert p_ref == p_port


def _launch(*extra):
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--selftest-launcher",
                           *extra], capture_output=True, text=True, timeout=300, cwd=ROOT)


def test_self_launcher_weak_two_ranks():
    # `bench.py --gpus 2` outside torchrun spawns 2 ranks itself (gloo here)
    out = _launch("--gpus", "2", "--steps", "3")
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["comm"]["world_size"] == 2
    assert line["ms_max"] == 11.0                                  # max over ranks
    assert [r["n_streams"] for r in line["per_rank"]] == [64, 64]
    assert [r["stream_id_sum"] for r in line["per_rank"]] == [sum(range(64)),
                                                             sum(range(64, 128))]
    assert line["value"] == pytest.approx(128 * 9 * 3 / 0.011, rel=1e-6)


def test_self_launcher_strong_sharding():
    out = _launch("--gpus", "4", "--scaling", "strong", "--streams", "10", "--steps", "2")
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["scaling"] == "strong" and line["n_gpus"] == 4
    assert [r["n_streams"] for r in line["per_rank"]] == [3, 3, 2, 2]     # stream_id % 4
    assert sum(r["stream_id_sum"] for r in line["per_rank"]) == sum(range(10))
    assert line["value"] == pytest.approx(10 * 9 * 2 / 0.013, rel=1e-6)


def test_world_size_mismatch_refused():
    import os
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode != 0 and "refusing" in out.stderr


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
