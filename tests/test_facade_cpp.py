"""The reference's OWN unit suites, compiled unchanged against the B200 façade.

tests/cpp/build.sh compiles /root/reference/proj/tests/{test_lora,
test_batch_select,test_workload}.cpp (read in place) against include/fusim/*.hpp
with a doctest-compatible shim and links them to libfusim_b200.so + libmlora.so.
test_batch_select / test_workload are host-only (MinPad packer, workload
cursor, seeded generators) and run here; test_lora's compute cases run the
façade's fused_forward / lora_forward / matmul on the GPU.
"""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "cpp", "build")


def _binary(name):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        if os.path.isdir("/root/reference/proj/tests"):
            subprocess.run(["bash", os.path.join(HERE, "cpp", "build.sh")], check=True)
        else:
            pytest.skip(f"{name} not built and /root/reference absent")
    return path


def _run(name):
    r = subprocess.run([_binary(name)], capture_output=True, text=True, timeout=600)
    summary = [ln for ln in r.stdout.splitlines() if ln.startswith("[doctest-shim]")]
    assert r.returncode == 0, r.stdout + r.stderr
    assert summary and "| 0 failed |" in summary[-1], summary
    return summary[-1]


def test_reference_batch_select_suite_on_facade():
    assert "15 passed" in _run("test_batch_select")


def test_reference_workload_suite_on_facade():
    assert "11 passed" in _run("test_workload")


@pytest.mark.gpu
def test_facade_fused_forward_bitwise_equals_reference_gpu():
    """fusim::fused_forward on the façade (device fp64, reference operation
    order) reproduces the reference's own outputs (tests/golden/, produced by
    the reference sources) BIT FOR BIT on all 66 golden instances."""
    import numpy as np

    from oracle.golden import unpack_case
    z = np.load(os.path.join(HERE, "golden", "lora_ref.npz"))
    keys = [str(k) for k in z["_index_forward"]]
    buf = [np.array([len(keys)], np.int32).tobytes()]
    for key in keys:
        W0, ranks, As, Bs, seqs = unpack_case(z, key)
        d, k = W0.shape
        buf.append(np.array([d, k, len(ranks), *ranks, len(seqs), *[j for j, _ in seqs],
                             *[x.shape[0] for _, x in seqs]], np.int32).tobytes())
        buf += [np.ascontiguousarray(W0).tobytes(), z[key + "A_all"].tobytes(), z[key + "B_all"].tobytes(),
                z[key + "X_all"].tobytes()]
    r = subprocess.run([_binary("facade_forward_io")], input=b"".join(buf), capture_output=True, timeout=600)
    assert r.returncode == 0, r.stderr.decode()
    got = np.frombuffer(r.stdout, np.float64)
    off = 0
    for key in keys:
        ref_out = z[key + "out"].ravel()
        assert np.array_equal(got[off:off + ref_out.size].view(np.uint64), ref_out.view(np.uint64)), key
        off += ref_out.size
    assert off == got.size


@pytest.mark.gpu
def test_reference_lora_suite_on_facade_gpu():
    # all 15 cases of test_lora.cpp, including "fused forward equals per-job
    # forward on real tokens" (100 trials, < 1e-9) and the BITWISE padding-
    # neutrality check, with the arithmetic on the device
    assert "15 passed" in _run("test_lora")


def test_reference_memory_model_suite_on_facade():
    # the reference's own test_memory_model.cpp (fit, NNLS, clamping, packing,
    # warm-up plan) against the product's memory model (facade_memory_model.cpp)
    assert "16 passed" in _run("test_memory_model")
