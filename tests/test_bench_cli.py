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


def test_gpus_flag_self_launches_one_process_per_gpu():
    """`bench.py --gpus N` with no launcher re-executes itself under
    torch.distributed.run (127.0.0.1 rendezvous): N processes, WORLD_SIZE = N."""
    env = dict(os.environ, MLORA_BENCH_PROBE_LAUNCH="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], capture_output=True,
                       text=True, timeout=180, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert all(x["world"] == 2 and x["gpus"] == 2 for x in lines)
    assert sorted(x["local_rank"] for x in lines) == [0, 1]


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", MLORA_BENCH_PROBE_LAUNCH="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], capture_output=True,
                       text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_launch_command_shape():
    sys.path.insert(0, ROOT)
    import bench
    cmd = bench.launch_command(8, ["--gpus", "8", "--steps", "20"], 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "20"]
