"""bench.py's multi-GPU launch contract on the CPU box: ``--gpus N`` must never silently time
fewer GPUs (it spawns N ranks itself, or checks torchrun's WORLD_SIZE), and fails loudly when the
GPUs are not there."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, **env):
    e = dict(os.environ, CUDA_VISIBLE_DEVICES="", **env)
    e.pop("WORLD_SIZE", None) if "WORLD_SIZE" not in env else None
    return subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True, timeout=300, cwd=ROOT,
                          env=e)


def test_gpus_without_devices_fails_loudly():
    out = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert out.returncode != 0
    assert "needs 2 GPUs" in out.stderr


def test_world_size_must_match_gpus():
    out = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"], WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    assert out.returncode != 0
    assert "WORLD_SIZE=1" in out.stderr


def test_reference_arm_on_non_zero_rank_exits_quietly():
    out = _run(["--impl", "reference", "--gpus", "2"], WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    assert out.returncode == 0 and out.stdout.strip() == ""
