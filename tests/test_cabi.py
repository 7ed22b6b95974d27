"""The drop-in boundary (CPU): libtgsx.so loads without a GPU, exports every function declared in
include/tgsx.h, the Python binding declares every one of them, and host-only entry points
work. No device compute is called here."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tgsx.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tgsx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for must in ("tgsx_render", "tgsx_backward", "tgsx_fit_step", "tgsx_densify",
                 "tgsx_view_accumulate", "tgsx_apply_step", "tgsx_budget_at"):
        assert must in fns


def test_library_exports_every_header_symbol():
    from paper_2412_13547_b200 import _lib
    path = _lib.LIB_PATH
    assert os.path.exists(path), "libtgsx.so not built"
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tgsx_[a-z0-9_]+)", out))
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    L = _lib.load()
    for f in header_functions():
        assert hasattr(L, f)
    assert set(header_functions()) <= set(_lib.SIGNATURES), set(header_functions()) - set(_lib.SIGNATURES)


def test_library_is_sm100a():
    from paper_2412_13547_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product():
    """The product never links or imports the checker."""
    pkg = os.path.join(ROOT, "paper_2412_13547_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                for bad in ("import oracle", "from oracle", "libtgs_oracle", "tgs_oracle.h",
                            "libtgs_ref", "oracle.bind", "or_render(", "or_backward("):
                    assert bad not in txt, (f, bad)
    out = subprocess.run(["ldd", os.path.join(pkg, "libtgsx.so")], capture_output=True, text=True).stdout
    assert "tgs_oracle" not in out and "tgs_ref" not in out


def test_host_entry_points_without_gpu():
    from paper_2412_13547_b200 import _lib
    L = _lib.load()
    st = (C.c_uint64 * 2)()
    L.tgsx_pcg32_init(st, 1, 1)
    u = L.tgsx_pcg32_uniform(st)
    assert 0.0 <= u < 1.0
    assert L.tgsx_budget_t_norm(300, 300, 3000) == 1.0
    assert L.tgsx_budget_t_norm(3000, 300, 3000) == 100.0
    h = C.c_void_p()
    assert L.tgsx_budget_create(10.0, 20.0, C.byref(h)) == 0
    assert L.tgsx_budget_at(h, 100.0) == 20
    L.tgsx_budget_destroy(h)


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-device error path")
def test_no_device_fails_loudly():
    from paper_2412_13547_b200 import _lib
    L = _lib.load()
    h = C.c_void_p()
    assert L.tgsx_create(0, C.byref(h)) != 0
