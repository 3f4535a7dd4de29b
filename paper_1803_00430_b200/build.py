"""Build the in-tree C-ABI library ``libechoforge_b200.so`` for sm_100a.

    python -m paper_1803_00430_b200.build      (or __graft_entry__.build())

nvcc cross-compiles without a GPU.  ``-fmad=false`` keeps every f64
expression of the exact-parity paths (intersection, sampling, SH) free of
FMA contraction, matching the reference's numpy evaluation; kernels that
want FMAs (the f32 slab test) use explicit __fmaf_rn.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libechoforge_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cpp")))


def build(verbose: bool = False, force: bool = False, profile_phases: bool = False) -> str:
    srcs = sources()
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "echoforge_b200.h"))
    lib = LIB.replace(".so", "_prof.so") if profile_phases else LIB
    if not force and os.path.exists(lib):
        t = os.path.getmtime(lib)
        if all(os.path.getmtime(d) <= t for d in deps):
            return lib
    cmd = [nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-ffp-contract=off",
           "-shared", "-o", lib + ".tmp", *srcs, "-lcudart"]
    if profile_phases:
        cmd.insert(1, "-DEF_PROFILE_PHASES")
    if verbose:
        cmd.insert(-1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True, profile_phases="--profile-phases" in sys.argv))
