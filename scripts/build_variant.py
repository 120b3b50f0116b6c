#!/usr/bin/env python3
"""Build a product-library variant with one source recompiled under extra -D
flags (A/B experiments): python scripts/build_variant.py NAME SRC.cu -DFOO=1 ...
→ _scratch/lib_NAME.so (git-ignored; travels to the GPU box). Load it with
SA_LIB=_scratch/lib_NAME.so in the timing scripts."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_06446_b200 import build as B  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
# SRC may be a path outside csrc/ (an older copy of a product source): it then
# replaces the product source of the same basename given by --replaces=NAME.cu
rep = next((d.split("=", 1)[1] for d in defs if d.startswith("--replaces=")), None)
defs = [d for d in defs if not d.startswith("--replaces=")]
B.build(debug=False)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_dir = os.path.join(root, "_scratch")
os.makedirs(out_dir, exist_ok=True)
obj = os.path.join(out_dir, f"{name}_{os.path.basename(src)[:-3]}.o")
cc = B.nvcc()
src_path = src if os.path.isabs(src) else os.path.join(B.CSRC, src)
src = rep or os.path.basename(src)
r = subprocess.run([cc, *B.ARCH, *B.NVCC_FLAGS, *defs, "-c", src_path, "-o", obj],
                   capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
objs = [os.path.join(B.OBJ, os.path.basename(s)[:-3] + ".o") for s in B.sources(False)
        if os.path.basename(s) != src] + [obj]
lib = os.path.join(out_dir, f"lib_{name}.so")
r = subprocess.run([cc, *B.ARCH, "-shared", "-Xlinker", "-Bsymbolic", "-o", lib, *objs, "-lcudart"],
                   capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
print(lib)
