"""Build libfpsa.so in-tree with nvcc for sm_100a (python -m paper_2506_04648_b200.build)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["csrc/fpsa_attn.cu", "csrc/fpsa_attn_bf16.cu", "csrc/fpsa_quant.cu", "csrc/fpsa_metrics.cu",
           "csrc/fpsa_io.cu", "csrc/fpsa_host.cpp"]
HEADERS = ["csrc/sm100.cuh", "csrc/softmax.cuh", "csrc/fpsa_internal.h", "../include/fpsa.h"]
TARGET = os.path.join(HERE, "libfpsa.so")
NVCC_FLAGS = [
    "-shared", "-Xcompiler", "-fPIC", "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(TARGET):
        return False
    t = os.path.getmtime(TARGET)
    return all(os.path.getmtime(os.path.join(HERE, s)) <= t for s in SOURCES + HEADERS)


def build_trace(extra=(), name="libfpsa_trace.so") -> str:
    """Instrumented variant (-DFPSA_TRACE, cycle counters; tools/trace_attn.py), never loaded by the package."""
    target = os.path.join(HERE, name)
    subprocess.run([nvcc(), *NVCC_FLAGS, "-DFPSA_TRACE", *extra, *SOURCES, "-o", target], cwd=HERE, check=True)
    return target


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return TARGET
    cmd = [nvcc(), *NVCC_FLAGS, *SOURCES, "-o", TARGET]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, cwd=HERE, check=True)
    return TARGET


if __name__ == "__main__":
    if "--variant" in sys.argv:  # python -m ...build --variant NAME -DFOO=1 ...: in-tree libfpsa_NAME.so
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], [a for a in sys.argv[i + 2:] if a.startswith("-D")]
        target = os.path.join(HERE, f"libfpsa_{name}.so")
        subprocess.run([nvcc(), *NVCC_FLAGS, *defs, *SOURCES, "-o", target], cwd=HERE, check=True)
        print(target)
        sys.exit(0)
    if "--trace" in sys.argv:
        print(build_trace())
        if "--nomma" in sys.argv:  # timing experiment: tensor core idle (results invalid)
            print(build_trace(("-DFPSA_NO_MMA",), "libfpsa_trace_nomma.so"))
        sys.exit(0)
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(TARGET)
