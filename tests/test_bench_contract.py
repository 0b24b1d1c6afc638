"""bench.py's reference arm prints one JSON line with the contract's keys (CPU)."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--case", "sh03b-desk",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
                "cpu_baseline", "e2e", "impl"):
        assert key in d, key
    assert d["impl"] == "reference" and d["higher_is_better"] is False and d["unit"] == "s/step"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
    assert set(d["split_s"]) == {"str", "nl", "coll", "field", "axpy_shear"}


def test_multi_rank_launcher_spawns_ranks_under_plain_python():
    """`python bench.py --gpus 2` (no torchrun) relaunches itself as 2 ranks; rank 0
    alone prints the line (CPU/gloo self-test of the same launcher)."""
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--launcher-selftest",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] == 2.0 and d["nccl_debug"] == "INFO"


import pytest  # noqa: E402


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--dist-stepper"]])
def test_bench_line_on_gpu(extra):
    """The GPU arm prints one line with the contract's keys (tiny case; the rank
    step over the P2P transport at one rank with --dist-stepper)."""
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--case", "c1-tiny", "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline", "--no-fp64-variant", *extra], capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e", "split_s"):
        assert key in d, key
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    if extra:
        assert "gk_dist_step" in d["config"]["step"] and d["rank_memory"]["world"] == 1


@pytest.mark.gpu
def test_bench_multi_rank_path_end_to_end():
    """`python bench.py --gpus 2` through the same launcher the driver uses, with
    both ranks on the one GPU (GK_BENCH_SHARED_GPU=1: gloo rendezvous, P2P
    transport between the two processes): one line, n_gpus 2, max over ranks."""
    import os
    env = dict(os.environ, GK_BENCH_SHARED_GPU="1")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--case", "c1-tiny", "--steps", "3",
                          "--warmup", "3"], capture_output=True, text=True, timeout=900, env=env)
    assert res.returncode == 0, (res.stdout[-2000:], res.stderr[-3000:])
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and "gk_dist_step_p2p" in d["config"]["step"]
    assert d["rank_memory"]["world"] == 2 and d["split_s"]["comm"] is None and d["e2e"]["value"] > 0
