"""Build a measurement variant of librnn.so with extra -D flags on one source file (the other
objects are the regular build's), into build/variants/librnn_<name>.so; select it at run time
with RNN_LIB=<path>.  Example:
  python profiles/build_variant.py dhn512x2 dhn.cu -DH4_THREADS_CFG=512 -DH4_CTAS_CFG=2 ..."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_24207_b200 import build as B  # noqa: E402

name, src, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
out_dir = os.path.join(ROOT, "build", "variants")
os.makedirs(out_dir, exist_ok=True)
obj = os.path.join(out_dir, f"{name}_{src}.o")
r = subprocess.run([B._nvcc(), *B.FLAGS, *flags, "-c", os.path.join(B.CSRC, src), "-o", obj],
                   capture_output=True, text=True)
assert r.returncode == 0, r.stderr
objs = [o for o in glob.glob(os.path.join(B.OBJ, "*.o")) if os.path.basename(o) != src + ".o"]
lib = os.path.join(out_dir, f"librnn_{name}.so")
r = subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-cudart", "shared", "-Xlinker",
                    "-rpath=/usr/local/cuda/lib64", "-o", lib, obj, *objs], capture_output=True,
                   text=True)
assert r.returncode == 0, r.stderr
print(lib)
