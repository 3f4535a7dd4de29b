"""Build the in-tree C-ABI library ``libechoforge_b200.so`` for sm_100a.

    python -m paper_1803_00430_b200.build      (or __graft_entry__.build())

nvcc cross-compiles without a GPU.  Every source compiles to its own object
in parallel (the trace kernels are split by family into
ef_trace_{brute,bvh}_nb{4,8}.cu for that), then one link.  ``-fmad=false``
keeps every f64 expression of the exact-parity paths (intersection,
sampling, SH) free of FMA contraction, matching the reference's numpy
evaluation; kernels that want FMAs (the f32 slab test) use explicit
__fmaf_rn.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libechoforge_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC,-ffp-contract=off"]
LIBS = ["-lcudart", "-ldl"]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cpp")))


def compile_library(out: str, extra=(), verbose: bool = False, jobs: int | None = None) -> str:
    """Compile every source (in parallel) with `extra` nvcc flags and link
    `out`; returns out."""
    nvcc = nvcc_path()
    srcs = sources()
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 1))
    with tempfile.TemporaryDirectory(prefix="ef_build_") as tmp:
        def one(src):
            obj = os.path.join(tmp, os.path.basename(src) + ".o")
            cmd = [nvcc, *ARCH, *FLAGS, *extra, "-c", "-o", obj, src]
            if verbose:
                cmd.insert(-4, "-Xptxas=-v")
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
            return obj
        with ThreadPoolExecutor(jobs) as ex:
            objs = list(ex.map(one, srcs))
        subprocess.check_call([nvcc, *ARCH, "-shared", "-o", out + ".tmp", *objs, *LIBS])
    os.replace(out + ".tmp", out)
    return out


def build(verbose: bool = False, force: bool = False, profile_phases: bool = False) -> str:
    srcs = sources()
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "echoforge_b200.h"))
    lib = LIB.replace(".so", "_prof.so") if profile_phases else LIB
    if not force and os.path.exists(lib):
        t = os.path.getmtime(lib)
        if all(os.path.getmtime(d) <= t for d in deps):
            return lib
    return compile_library(lib, ["-DEF_PROFILE_PHASES"] if profile_phases else [], verbose=verbose)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True, profile_phases="--profile-phases" in sys.argv))
