"""The C ABI from a plain C11 host program (tests/c_abi/train_step.c): no
Python or torch between the caller and libmlora.so.  CPU: the header is valid
C and the program compiles and links against the in-tree library.  GPU: it runs
pack -> forward -> backward -> AdamW on cuda:0 and checks every result against
its own fp64 CPU computation."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2312_02515_b200")
SRC = os.path.join(ROOT, "tests", "c_abi", "train_step.c")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _compile(out: str) -> None:
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    if not os.path.exists(os.path.join(PKG, "libmlora.so")):
        pytest.fail("libmlora.so is not built (python -c 'import __graft_entry__ as g; g.build()')")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), SRC, "-L", PKG, "-lmlora", f"-Wl,-rpath,{PKG}",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_c_program_compiles_and_links(tmp_path):
    _compile(str(tmp_path / "train_step"))


@pytest.mark.gpu
def test_c_program_trains_one_step(tmp_path):
    exe = str(tmp_path / "train_step")
    _compile(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("OK")
    assert r.stdout.count(" ok") >= 9  # Y, dX, dA, dB per job + AdamW
