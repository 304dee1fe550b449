"""Build libbh.so in-tree with nvcc for sm_100a (no GPU needed).

    python -m paper_2203_08966_b200.build_lib

bh_exact.cu is compiled with -fmad=false (reference fp64 arithmetic never
contracts multiply-adds); the other units use the default contraction.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libbh.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE,
          "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
UNITS = {
    "bh_exact.cu": ["-fmad=false"],
    "bh_fast.cu": [],
    "bh_sort.cu": [],
    "bh_walk.cu": ["-ftz=true"],
    "bh_api.cu": [],
    "bh_host.cpp": ["-Xcompiler", "-ffp-contract=off", "-x", "cu"],
}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cuh", ".h", ".cpp"))] + [os.path.join(INCLUDE, "bh.h")]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    cc = nvcc()
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for unit, extra in UNITS.items():
        obj = os.path.join(objdir, os.path.splitext(unit)[0] + ".o")
        cmd = [cc, *ARCH, *COMMON, *extra, "-c", os.path.join(CSRC, unit), "-o", obj]
        cmd += os.environ.get("BH_NVCC_EXTRA", "").split()
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = OUT + ".tmp"
    subprocess.run([cc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt",
                    "-lpthread", "-ldl"], check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv))
