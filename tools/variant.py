"""A/B experiment builds: compiles libtgsx.so with extra nvcc flags into exp/<name>/libtgsx.so
(git-ignored, travels to the GPU box with the snapshot). Select one at run time with
TGSX_LIB=exp/<name>/libtgsx.so. Usage: python tools/variant.py NAME [-DFOO=1 ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_13547_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "exp", name)
os.makedirs(out, exist_ok=True)
b.OBJ = os.path.join(out, "obj")
b.LIB = os.path.join(out, "libtgsx.so")
print(b.build(extra=flags, force=True))
