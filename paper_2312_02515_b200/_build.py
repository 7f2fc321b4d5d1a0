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

MLORA_SOURCES = ["mlora_capi.cu", "mlora_f64.cu", "mlora_model.cu", "mlora_decoder.cu", "mlora_layer.cu", "mlora_comm.cpp"]
MLORA_HEADERS = ["sm100.cuh", "mlora_gemm.cuh", "mlora_aux.cuh", "mlora_down_multi.cuh"]
FACADE_SOURCES = ["facade_lora.cpp", "facade_batch_select.cpp", "facade_workload.cpp", "facade_capi.cpp",
                  "facade_memory_model.cpp",
                  "facade_b200.cpp"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps if os.path.exists(d))


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


OBJ_DIR = os.path.join(PKG, "build")
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3"]


def _compile_one(src: str, deps: list[str], force: bool) -> str:
    """One translation unit -> build/<name>.o, skipped when newer than its deps."""
    obj = os.path.join(OBJ_DIR, os.path.basename(src) + ".o")
    if force or not _newer(obj, [src, *deps]):
        _run([NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj])
    return obj


def build_mlora(force: bool = False) -> str:
    """libmlora.so: every .cu / .cpp compiled in parallel (one nvcc per TU, each
    object cached by mtime), then one link.  The CUDA runtime is linked
    statically here and ONLY here: the façade goes through this library's
    mlora_malloc / mlora_memcpy, so a process holds one runtime instance."""
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ_DIR, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in MLORA_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    hdrs = [os.path.join(CSRC, h) for h in MLORA_HEADERS] + [os.path.join(ROOT, "include", "mlora.h")]
    with ThreadPoolExecutor(len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile_one(s, hdrs, force), srcs))
    if not force and _newer(LIB_MLORA, objs):
        return LIB_MLORA
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB_MLORA, *objs, "-ldl"])
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
    # no CUDA runtime here: device memory, copies and syncs go through libmlora.so
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", inc, "-o", LIB_FACADE, *srcs, "-L", PKG,
           "-lmlora", "-Wl,-rpath,$ORIGIN", "-lpthread"]
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
