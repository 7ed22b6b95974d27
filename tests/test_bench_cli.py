"""bench.py contract pieces that run without a GPU: argument handling and the reference arm of
the configs the reference cannot run (the 3-D front end has no reference counterpart)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=120, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    return [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]


def test_reference_arm_3d_configs_report_unavailable():
    for cfg in ("c6", "c7", "c9"):
        lines = _run("--impl", "reference", "--config", cfg)
        assert len(lines) == 1
        assert lines[0]["impl"] == "reference" and "unavailable" in lines[0]


def test_help_lists_configs():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True,
                         text=True, timeout=60, cwd=ROOT)
    assert out.returncode == 0
    for cfg in ("c2", "c3", "c4", "c5", "c6", "c7", "c8", "c9"):
        assert cfg in out.stdout


def test_gpus_flag_launches_that_many_ranks():
    """`bench.py --gpus 2` (the driver's command form, no torchrun around it) starts 2 ranks
    itself under torch.distributed.run; --launch-check makes each rank report and exit."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"],
                         capture_output=True, text=True, timeout=180, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert sorted((d["rank"], d["world"]) for d in lines) == [(0, 2), (1, 2)]


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"],
                         capture_output=True, text=True, timeout=60, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)
