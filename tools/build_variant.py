"""Build a tuning variant of the library with extra nvcc -D flags into
paper_2202_10297_b200/_lib/var_<name>.so (objects under build/var_<name>/).
Used only by timing experiments (tools/time_variants.py); the product is the
default build.   python tools/build_variant.py NAME -DX=1 [-DY=2 ...]"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_10297_b200 import _build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
obj_dir = os.path.join(B.ROOT, "build", "var_" + name)
out = os.path.join(B.PKG, "_lib", "var_" + name + ".so")
os.makedirs(obj_dir, exist_ok=True)
srcs = sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))


def comp(src):
    o = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
    r = subprocess.run([B.NVCC] + B.FLAGS + defs + ["-c", src, "-o", o], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return o


with cf.ThreadPoolExecutor(os.cpu_count() or 4) as ex:
    objs = list(ex.map(comp, srcs))
r = subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-cudart", "static", "-o", out] + objs + ["-ldl"],
                   capture_output=True, text=True)
if r.returncode:
    raise RuntimeError(r.stderr)
print(out)
