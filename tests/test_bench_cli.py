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
    for cfg in ("c6", "c7"):
        lines = _run("--impl", "reference", "--config", cfg)
        assert len(lines) == 1
        assert lines[0]["impl"] == "reference" and "unavailable" in lines[0]


def test_help_lists_configs():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True,
                         text=True, timeout=60, cwd=ROOT)
    assert out.returncode == 0
    for cfg in ("c2", "c3", "c4", "c5", "c6", "c7"):
        assert cfg in out.stdout
