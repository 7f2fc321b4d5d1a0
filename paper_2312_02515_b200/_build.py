"""Build the in-tree native libraries with nvcc / g++ (no JIT cache).

``libmlora.so``       the sm_100a kernels + C ABI (include/mlora.h)
``libfusim_b200.so``  the C++ façade reproducing fusim/lora.hpp over the C ABI

Both land next to this file so they travel with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

LIB_MLORA = os.path.join(PKG, "libmlora.so")
LIB_FACADE = os.path.join(PKG, "libfusim_b200.so")

MLORA_SOURCES = ["mlora_capi.cu", "mlora_f64.cu", "mlora_model.cu", "mlora_decoder.cu", "mlora_comm.cpp"]
MLORA_HEADERS = ["sm100.cuh", "mlora_gemm.cuh", "mlora_aux.cuh", "mlora_quad.cuh", "mlora_down_multi.cuh"]
FACADE_SOURCES = ["facade_lora.cpp", "facade_batch_select.cpp", "facade_workload.cpp", "facade_capi.cpp"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps if os.path.exists(d))


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build_mlora(force: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in MLORA_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    deps = srcs + [os.path.join(CSRC, h) for h in MLORA_HEADERS] + [os.path.join(ROOT, "include", "mlora.h")]
    if not force and _newer(LIB_MLORA, deps):
        return LIB_MLORA
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
           "-cudart", "static", "-I", os.path.join(ROOT, "include"), "-o", LIB_MLORA, *srcs, "-ldl"]
    _run(cmd)
    return LIB_MLORA


def build_facade(force: bool = False) -> str | None:
    srcs = [os.path.join(CSRC, s) for s in FACADE_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if not srcs:
        return None
    inc = os.path.join(ROOT, "include")
    fdir = os.path.join(inc, "fusim")
    deps = srcs + [LIB_MLORA] + ([os.path.join(fdir, h) for h in os.listdir(fdir)] if os.path.isdir(fdir) else [])
    if not force and _newer(LIB_FACADE, deps):
        return LIB_FACADE
    cuda = os.path.dirname(os.path.dirname(NVCC))
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", inc, "-I", os.path.join(cuda, "include"),
           "-o", LIB_FACADE, *srcs, "-L", PKG, "-lmlora", "-Wl,-rpath,$ORIGIN",
           "-L", os.path.join(cuda, "lib64"), "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    _run(cmd)
    return LIB_FACADE


def build_cpp_tests() -> None:
    """The reference's own unit suites compiled against the façade (needs /root/reference)."""
    script = os.path.join(ROOT, "tests", "cpp", "build.sh")
    if os.path.exists(script):
        _run(["bash", script])


def build_all(force: bool = False) -> None:
    build_mlora(force)
    build_facade(force)
    build_cpp_tests()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
