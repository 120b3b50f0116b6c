"""Build libshiftadd_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2306_06446_b200.build [--force] [--verbose]

Object files go to paper_2306_06446_b200/_build/, the shared library next to
this file. No fast-math / FTZ: the sign-hash and router must see negative
subnormals and exact float32 rounding.

Two libraries are built from the same sources:
- libshiftadd_b200.so (the product): kernel-variant switches are compile-time
  constants, no probe kernels;
- libshiftadd_b200_debug.so (-DSA_DEBUG, + the MMA-rate probes of
  tc_probe.cu): the sa_debug_* setters the A/B tests and scripts/ use.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libshiftadd_b200.so")
DEBUG_LIB = os.path.join(HERE, "libshiftadd_b200_debug.so")
# diagnostics kernels and measured-and-reverted variants: never in the product library
DEBUG_ONLY = ("tc_probe.cu", "binattn_stream.cu")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-warn-spills", "-I", INCLUDE, "-I", CSRC]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources(debug=False):
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith(".cu") and (debug or f not in DEBUG_ONLY))


def _deps_mtime():
    paths = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    paths += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    paths.append(os.path.abspath(__file__))
    return max(os.path.getmtime(p) for p in paths)


def up_to_date(lib=LIB) -> bool:
    return os.path.exists(lib) and os.path.getmtime(lib) >= _deps_mtime()


def build(force: bool = False, verbose: bool = False, debug: bool = True) -> str:
    """Build the product library and (unless debug=False) the debug library."""
    if debug:
        with cf.ThreadPoolExecutor(max_workers=2) as ex:
            futs = [ex.submit(_build_one, force, verbose, False),
                    ex.submit(_build_one, force, verbose, True)]
            return [f.result() for f in futs][0]
    return _build_one(force, verbose, False)


def _build_one(force: bool, verbose: bool, debug: bool) -> str:
    lib_path = DEBUG_LIB if debug else LIB
    if not force and up_to_date(lib_path):
        return lib_path
    obj_dir = os.path.join(OBJ, "debug") if debug else OBJ
    os.makedirs(obj_dir, exist_ok=True)
    flags = NVCC_FLAGS + (["-DSA_DEBUG"] if debug else [])
    cc = nvcc()
    hdr_mtime = max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC)
                    if f.endswith((".cuh", ".h")))
    hdr_mtime = max(hdr_mtime, max(os.path.getmtime(os.path.join(INCLUDE, f))
                                   for f in os.listdir(INCLUDE)))

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
                os.path.getmtime(src), hdr_mtime):
            return obj, ""
        cmd = [cc, *ARCH, *flags, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, sources(debug)))
    for _, log in results:
        if verbose and log.strip():
            print(log, file=sys.stderr)
    objs = [o for o, _ in results]
    tmp = lib_path + ".tmp"
    # -Bsymbolic: the product and debug libraries define the same template
    # kernels; each must launch its own (a test process loads both)
    cmd = [cc, *ARCH, "-shared", "-Xlinker", "-Bsymbolic", "-Xlinker", "--no-undefined", "-o", tmp,
           *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib_path)
    return lib_path


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    main()
