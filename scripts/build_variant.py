"""Build an experimental libsbr200 variant with extra -D flags into
build_variants/<name>.so (select it at run time with SBR_LIB=...).
  python scripts/build_variant.py NAME -DSBR_TRACE_MINB=6 ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_09243_b200 import _build as B
name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "build_variants")
os.makedirs(os.path.join(out_dir, name), exist_ok=True)
objs = []
procs = []
for src in B.SOURCES:
    obj = os.path.join(out_dir, name, os.path.splitext(src)[0] + ".o")
    procs.append(subprocess.Popen([B.nvcc(), *B.ARCH, *B.NVCC_FLAGS, *defs, "-c",
                                   os.path.join(B.CSRC, src), "-o", obj]))
    objs.append(obj)
assert all(p.wait() == 0 for p in procs)
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", os.path.join(out_dir, name + ".so"), *objs,
                "-lcudart"], check=True)
print(os.path.join(out_dir, name + ".so"))
