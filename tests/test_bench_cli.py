"""bench.py's contract on the host side (no GPU): the reference arm of the
model-level config reports `unavailable` (the reference has no model), the
config table covers the BASELINE configs the bench measures, and the CLI parses."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=120, cwd=ROOT)


def test_reference_arm_of_decoder_config_is_unavailable():
    r = run("--impl", "reference", "--config", "c4")
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and "unavailable" in line


def test_config_table():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.CONFIGS["c2"]["ranks"] == [16] * 4 and bench.CONFIGS["c2"]["seqs"] * bench.CONFIGS["c2"]["seq_len"] == 2048
    assert len(bench.CONFIGS["c5"]["ranks"]) == 32 and bench.CONFIGS["c5"]["jobs_total"]
    assert bench.CONFIGS["c4"]["decoder"] == "chatglm2-6b" and len(bench.CONFIGS["c4"]["ranks"]) == 6


def test_help():
    r = run("--help")
    assert r.returncode == 0 and "--config" in r.stdout


def test_default_steps_cover_the_nvml_refresh():
    """Without --steps each config times about 1 s of device work (NVML refreshes
    clocks / reasons / power about every 100 ms), and every config has a default."""
    sys.path.insert(0, ROOT)
    import bench
    assert set(bench.DEFAULT_STEPS) == set(bench.CONFIGS)
    ms_per_step = {"c2": 5.2, "c5": 42.0, "c4": 300.0}  # measured on one B200 (profiles/)
    for name, steps in bench.DEFAULT_STEPS.items():
        assert steps * ms_per_step[name] >= 1000.0, name
