"""The product's interval box mask (csrc/tgsx_device.cuh box_mask, used by the forward and the
backward to build the per-tile pass matrix) equals the per-column box test of
rasterizer.cpp:116-118 bit for bit on 2^28 hashed cases, including boxes whose edges sit exactly
on, or one ulp beside, active pixel centres (tests/cuda/box_mask_check.cu)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "paper_2412_13547_b200", "csrc")


def test_interval_box_mask_is_exact(tmp_path):
    exe = str(tmp_path / "box_mask_check")
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "--expt-relaxed-constexpr", f"-I{CSRC}", os.path.join(HERE, "cuda", "box_mask_check.cu"),
                    "-o", exe], check=True, capture_output=True)
    r = subprocess.run([exe, "28"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches 0" in r.stdout
