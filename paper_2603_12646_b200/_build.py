"""nvcc build recipe for librf_fa.so (in-tree, sm_100a only).

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.  nvcc
cross-compiles without a GPU, so this also runs on the CPU-only dev container.
"""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librf_fa.so")
SOURCES = ["fa_fwd_sm100.cu", "fa_fwd_sm100_d128.cu", "fa_fwd_sm100_local.cu", "fa_fwd_simt.cu", "fa_aux.cu", "fa_api.cu", "encoder_ops.cu", "gemm_sm100.cu", "clf_runtime.cu", "host_cast.cpp",
           # graph layer around the operator: IR, SDPA -> FusedFlashAttention rewriter, GPU executor, C ABI
           os.path.join("graph", "graph_ir.cpp"), os.path.join("graph", "sdpa_rewriter.cpp"),
           os.path.join("graph", "graph_executor.cu"), os.path.join("graph", "graph_capi.cpp")]
INCLUDE = os.path.normpath(os.path.join(HERE, "..", "include"))
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177", "-I", INCLUDE, "-ldl",
]
HEADERS = ["ptx.cuh", "fa_internal.h", "host_cast.h", os.path.join("graph", "json.hpp"),
           os.path.join(INCLUDE, "rf_fa.h"), os.path.join(INCLUDE, "rf_graph.h"), os.path.join(INCLUDE, "rf_clf.h"), os.path.join(INCLUDE, "rf_gemm.h"),
           os.path.join(INCLUDE, "routefast_b200", "attention.hpp"), os.path.join(INCLUDE, "routefast_b200", "graph.hpp"),
           os.path.join(INCLUDE, "routefast_b200", "classifiers.hpp")]




def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build librf_fa.so")


def sources() -> list:
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def is_stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every CUDA source into paper_2603_12646_b200/librf_fa.so."""
    if not force and not is_stale():
        return LIB
    cmd = [nvcc_path()] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-o", LIB] + sources()
    env = dict(os.environ)
    # the image exports CC/CXX pointing at a wrapper without spec files; let nvcc use the system g++
    env.pop("CC", None)
    env.pop("CXX", None)
    res = subprocess.run(cmd, capture_output=True, text=True, env=env)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stderr)
    return LIB


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))


def build_variant(name: str, defines: dict) -> str:
    """Developer aid: an experimental build of the same ABI with -D overrides (kernel tuning);
    select it at run time with RF_FA_LIB=<path>."""
    out = os.path.join(HERE, f"librf_fa_{name}.so")
    cmd = [nvcc_path()] + NVCC_FLAGS + [f"-D{k}={v}" for k, v in defines.items()] + ["-o", out] + sources()
    env = dict(os.environ)
    env.pop("CC", None)
    env.pop("CXX", None)
    res = subprocess.run(cmd, capture_output=True, text=True, env=env)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    return out
