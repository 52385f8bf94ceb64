"""Build an A/B variant of libgsr.so with extra nvcc defines:
python tools/build_variant.py TAG -DNAME=VALUE ...  ->  paper_2408_12677_b200/libgsr_TAG.so
(load it with GSR_LIB=libgsr_TAG.so)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12677_b200 import _build  # noqa: E402

tag, defines = sys.argv[1], sys.argv[2:]
objdir = os.path.join(_build.PKG, "build", "var_" + tag)
os.makedirs(objdir, exist_ok=True)
objs = []
for s in _build.SOURCES:
    o = os.path.join(objdir, os.path.splitext(s)[0] + ".o")
    _build._compile(s, o, defines)
    objs.append(o)
subprocess.check_call([_build.nvcc(), *_build.ARCH, "-shared", "-o", os.path.join(_build.PKG, f"libgsr_{tag}.so"), *objs])
print("built", f"libgsr_{tag}.so")
