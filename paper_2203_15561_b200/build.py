"""In-tree build of the sm_100a extension (explicit nvcc; no JIT cache).

Produces paper_2203_15561_b200/_genasm.so: the fused DC+TB kernel, the C-ABI
host side and the workload generator, cudart linked statically so the .so
loads on the GPU box without a toolkit path.  check=True builds the same
library with the kernel's contract checks (-DGA_CHECK, the PrunedAccess /
bounds tripwires) into _genasm_check.so, for tests/test_check_build.py.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "_genasm.so")
CHECK_SO = os.path.join(HERE, "_genasm_check.so")
SOURCES = ["genasm_lockstep.cu", "genasm_thread.cu", "genasm_capi.cu", "genasm_pack.cu", "sim.cpp",
           "accounting.cpp", "microbench.cu", "genasm_io.cpp", "genasm_baseline.cu", "genasm_dp.cu", "pack_host.cpp"]
HEADERS = ["genasm_kernel.cuh", "genasm_device.cuh", "genasm_thread.cuh", "../../include/genasm.h",
           "../../include/genasm_sim.h", "../../include/genasm_bench.h", "../../include/genasm_io.h"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-O3,-pthread", "-Xptxas", "-v", "-shared", "-cudart", "static"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build(so: str = SO) -> bool:
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, check: bool = False) -> str:
    so = CHECK_SO if check else SO
    if not force and not needs_build(so):
        return so
    srcs = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    cmd = [_nvcc(), *NVCC_FLAGS, *(["-DGA_CHECK"] if check else []), "-o", so + ".tmp", *srcs]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"nvcc failed building {os.path.basename(so)}")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(so + ".tmp", so)
    return so


def outcomes_so() -> str:
    import sysconfig
    return os.path.join(HERE, "_outcomes" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))


def build_outcomes(force: bool = False) -> str:
    """The CPython extension that builds the drop-in API's result objects in
    bulk (csrc/outcomes_py.cpp; host code, g++ against this interpreter)."""
    import sysconfig
    so = outcomes_so()
    src = os.path.join(CSRC, "outcomes_py.cpp")
    if not force and os.path.exists(so) and os.path.getmtime(so) >= os.path.getmtime(src):
        return so
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-shared", "-fPIC",
           "-I" + sysconfig.get_paths()["include"], "-o", so + ".tmp", src]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("g++ failed building _outcomes")
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, check="--check" in sys.argv)
    build_outcomes(force="--force" in sys.argv)
