#!/usr/bin/env python
"""bench.py — effective (non-pad) tokens/s of the fused multi-LoRA fwd+bwd step.

Metric (BASELINE.json): effective tokens/s, LLaMA-7B-shaped layer, 4 fused LoRA
jobs.  One "step" = one fused training iteration of one LLaMA-7B layer's seven
LoRA'd projections (q, k, v, o, gate, up, down) over one fused batch: every
forward, the per-job loss, every backward (dX, dA_j, dB_j) and one per-job-lr
AdamW update (paper_2312_02515_b200/layer.py).  Config C2: 4 jobs x rank 16,
lr = {1e-4, 2e-4, 5e-5, 3e-4}, batch 4 x 512 tokens per job -> 8192 effective
tokens per step per GPU (δ = 0).  Synthetic data, random-init weights.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): adapter-parallel weak scaling — each
rank owns 4 jobs (32 jobs at N=8), the frozen base weights are
broadcast once from rank 0 over NCCL at init, and the steady state has no
collective.  Time = max over ranks of the CUDA-event time of the K steps.

`--impl reference` times the reference's own CPU fused_forward
(/root/reference/proj/src/lora.cpp:160-182, compiled in place into
oracle/_ref/libfusim_ref.so) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective (non-pad) tokens/sec, LLaMA-7B shape, 4 fused LoRA jobs, 1-8 GPU"
UNIT = "tokens/s"

DEFAULT_STEPS = {"c2": 200, "c5": 30, "c4": 5}  # ~1.0 s, ~1.3 s, ~1.5 s of device time on one B200

CONFIGS = {
    # name: (shape set, ranks, lrs, sequences per job, tokens per sequence)
    "c2": dict(shapes="llama7b", ranks=[16, 16, 16, 16], lrs=[1e-4, 2e-4, 5e-5, 3e-4], seqs=4, seq_len=512,
               workload="llama7b-layer(q,k,v,o,gate,up,down) x 4 jobs r16, batch 4x512/job, fwd+bwd+AdamW"),
    # BASELINE C5: 32 jobs in total on LLaMA-7B shapes, partitioned across the N GPUs
    # (strong scaling in jobs: 32 / N jobs, 32 / N x 2048 tokens per GPU per step)
    "c5": dict(shapes="llama7b", ranks=[16] * 32, lrs=[1e-4, 2e-4, 5e-5, 3e-4] * 8, seqs=4, seq_len=512,
               jobs_total=True,
               workload="llama7b-layer(q,k,v,o,gate,up,down) x 32 jobs r16 in total (partitioned over the GPUs), "
                        "batch 4x512/job, fwd+bwd+AdamW"),
    # model level (not the headline): BASELINE C4, the whole ChatGLM2-6B-shaped decoder
    "c4": dict(decoder="chatglm2-6b", ranks=[16] * 6, lrs=[1e-4, 2e-4, 5e-5, 3e-4, 1e-4, 2e-4], seqs=4,
               seq_len=512, workload="chatglm2-6b decoder (28 layers, MQA, V 65024) x 6 jobs r16, batch 4x512/job, "
                                     "fwd + per-job masked CE + bwd + AdamW"),
}
DECODER_METRIC = "effective (non-pad) tokens/sec, ChatGLM2-6B decoder, 6 fused LoRA jobs (model level, BASELINE C4)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(bf16=d["bf16_tflops"], bf16_sustained=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    hbm=d["hbm_gbs"], source="MEASURED_PEAKS.json")
    return dict(bf16=1590.0, bf16_sustained=1400.0, hbm=6650.0, source="fallback (B200_PROFILING.md)")


# ----------------------------------------------------------------------------- clocks
REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x10: "sync_boost"}


class ClockSampler(threading.Thread):
    """Samples SM clock + throttle reasons through NVML while the timed region runs."""

    def __init__(self, torch_dev, period=0.005):
        super().__init__(daemon=True)
        self.period = period
        self.samples = []
        self.power = []
        self.power_limit_w = None
        self.reasons = 0
        self.max_mhz = None
        self._halt = threading.Event()
        self.ok = False
        try:
            import pynvml as nv
            self.nv = nv
            nv.nvmlInit()
            import torch
            props = torch.cuda.get_device_properties(torch_dev)
            try:
                bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
                self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = nv.nvmlDeviceGetHandleByIndex(torch_dev.index or 0)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            try:
                self.power_limit_w = nv.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0
            except Exception:
                pass
            self.ok = True
        except Exception:
            pass

    def run(self):
        if not self.ok:
            return
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self._halt.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= get_reasons(self.h)
                self.power.append(self._power_w())
            except Exception:
                pass
            time.sleep(self.period)

    def _power_w(self):
        # instantaneous board power where the driver has it (GetPowerUsage is a ~1 s average)
        nv = self.nv
        fi = getattr(nv, "NVML_FI_DEV_POWER_INSTANT", None)
        if fi is not None:
            try:
                v = nv.nvmlDeviceGetFieldValues(self.h, [fi])[0]
                if v.nvmlReturn == 0:
                    return v.value.uiVal / 1000.0
            except Exception:
                pass
        return nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0

    def stop(self):
        self._halt.set()
        self.join(timeout=2)
        med = statistics.median(self.samples) if self.samples else None
        # board power (instantaneous) against the enforced limit shows the power cap
        # directly: the step is power-bound
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": [n for b, n in REASONS.items() if self.reasons & b],
                "power_w_median": statistics.median(self.power) if self.power else None,
                "power_w_max": max(self.power) if self.power else None,
                "power_limit_w": self.power_limit_w}


# ----------------------------------------------------------------------------- reference CPU arm
def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_sample(cfg, seq_len=64, seed=1, replicas=1):
    """Pre-marshalled reference fused_forward calls: `replicas` independent fused
    samples (J jobs x 1 sequence x seq_len tokens each) per projection of the
    layer, all sharing that projection's frozen W0.  Forward only: the reference
    has no backward."""
    import numpy as np
    from oracle import ref
    from paper_2312_02515_b200.layer import SHAPES
    rng = np.random.default_rng(seed)
    calls = []
    ranks = cfg["ranks"][:4]  # the reference loops per sequence: its cost per token does not depend on J
    J = len(ranks)
    for _, d, k, _ in SHAPES[cfg["shapes"]]:
        W0 = rng.uniform(-1, 1, (d, k)) / np.sqrt(k)
        w = ref.Weights(W0)
        del W0
        As = [rng.uniform(-1, 1, (r, k)) for r in ranks]
        Bs = [rng.uniform(-1, 1, (d, r)) for r in ranks]
        for _ in range(replicas):
            seqs = [(j, rng.uniform(-1, 1, (seq_len, k))) for j in range(J)]
            calls.append(ref.FusedCall(w, ranks, As, Bs, seqs))
    return calls, J * seq_len * replicas


def time_reference(cfg, steps, warmup, seq_len=64, budget_s=None):
    """Runs the reference's fused_forward on every host core: each step is
    `replicas` independent fused samples per projection of the layer, one
    single-threaded (reentrant) reference call per host thread.  With budget_s,
    stops taking timed steps once the budget is spent (at least one)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import ref
    if not ref.available():
        ref.build()
    if not ref.available():
        return None
    nproj = len(__import__("paper_2312_02515_b200.layer", fromlist=["SHAPES"]).SHAPES[cfg["shapes"]])
    replicas = max(1, min(8, host_threads() // nproj))
    calls, tokens = reference_sample(cfg, seq_len, replicas=replicas)
    threads = min(len(calls), host_threads())
    times = []
    t_start = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        for i in range(warmup + steps):
            if budget_s is not None and times and time.perf_counter() - t_start > budget_s:
                break
            t0 = time.perf_counter()
            list(ex.map(lambda c: c(), calls))
            dt = time.perf_counter() - t0
            if i >= warmup:
                times.append(dt)
    total = sum(times)
    return dict(value=tokens * len(times) / total, unit=UNIT, cores=threads, kind="reference",
                sample=f"reference fusim::fused_forward (fp64, forward only): {replicas} fused sample(s) of "
                       f"{min(4, len(cfg['ranks']))} jobs x 1 seq x {seq_len} tokens per LLaMA-7B projection x {nproj} "
                       f"projections = {tokens} effective tokens per step, {len(calls)} concurrent reference calls "
                       f"on {threads} host threads ({host_threads()} available); {len(times)} timed steps, {total:.1f} s",
                ms_per_step=1e3 * total / len(times), steps_run=len(times))


def time_reference_single_core(cfg, seq_len=16):
    """The reference's own path as it ships: ONE process, ONE thread
    (lora.cpp:160-182 is single-threaded).  One fused_forward
    call per projection of the layer, run back to back on one host thread, on a
    smaller sample than the all-core leg (J jobs x 1 seq x `seq_len` tokens per
    projection) so it stays ~15-20 s."""
    from oracle import ref
    if not ref.available():
        ref.build()
    if not ref.available():
        return None
    calls, tokens = reference_sample(cfg, seq_len, seed=2, replicas=1)
    t0 = time.perf_counter()
    for c in calls:
        c()
    dt = time.perf_counter() - t0
    return dict(value=tokens / dt, unit=UNIT, cores=1, kind="reference",
                sample=f"reference fusim::fused_forward (fp64, forward only), one process, one thread: "
                       f"{len(calls)} projections x {min(4, len(cfg['ranks']))} jobs x 1 seq x {seq_len} tokens "
                       f"= {tokens} effective tokens in {dt:.1f} s (host nproc = {os.cpu_count()}, "
                       f"affinity = {host_threads()})")


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps = max(1, args.steps)
    warmup = max(0, args.warmup)
    # the reference CPU path takes ~10 s per step: bound the arm to a few minutes
    r = time_reference(cfg, steps, warmup, budget_s=float(os.environ.get("MLORA_REF_BUDGET_S", "180")))
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfusim_ref.so not built and "
                          "/root/reference absent"}))
        return 0
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": r["steps_run"], "requested_steps": steps, "warmup": warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"] + " [reference CPU sample: see cpu_baseline.sample]"},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- our arm
def launch_command(gpus: int, argv: list[str], port: int) -> list[str]:
    """`python bench.py --gpus N ...` without a launcher re-executes itself under
    torch.distributed.run: one process per GPU, rendezvous on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def self_launch(gpus: int) -> int:
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    # NCCL's init log (rank count, transport) goes to stderr for the record
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = launch_command(gpus, sys.argv[1:], port)
    print("[bench] " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: about 1 s of device time per config; 30 for --impl reference)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None and int(env_world) != args.gpus and args.impl != "reference":
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={env_world}: launch one process per GPU "
              f"(torch.distributed.run --nproc-per-node {args.gpus}) or drop --gpus", file=sys.stderr)
        return 2
    if env_world is None and args.gpus > 1 and args.impl != "reference":
        return self_launch(args.gpus)
    if os.environ.get("MLORA_BENCH_PROBE_LAUNCH") == "1":  # CPU test of the launcher: report the rank layout
        print(json.dumps({"rank": int(os.environ.get("RANK", "0")), "world": int(os.environ.get("WORLD_SIZE", "1")),
                          "local_rank": int(os.environ.get("LOCAL_RANK", "0")), "gpus": args.gpus}), flush=True)
        return 0
    if args.steps is None:
        # NVML refreshes SM clocks / clock-event reasons / power about every 100 ms
        # (tools/nvml_probe.py), so the timed region defaults to about 1 s of device
        # time for the clock evidence to describe it
        args.steps = 30 if args.impl == "reference" else DEFAULT_STEPS[args.config]
    if "decoder" in cfg:
        return run_decoder(args, cfg)
    if args.impl == "reference":
        return run_reference_arm(args, cfg)

    import torch
    import torch.distributed as dist
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200.layer import SHAPES, FusedLoraLayer, flops_per_token

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one process per GPU.  (MLORA_BENCH_SHARE_GPU=1 folds ranks onto the visible
    # devices and uses gloo — only to exercise the multi-rank logic on a 1-GPU box.)
    share = os.environ.get("MLORA_BENCH_SHARE_GPU") == "1"
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if share:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_2312_02515_b200 import parallel as PL

    shapes = SHAPES[cfg["shapes"]]
    per_job = cfg["seqs"] * cfg["seq_len"]
    # adapter-parallel weak scaling: 4 jobs per GPU (32 jobs at N=8, C5), partitioned by LPT
    # weak scaling (default): the config's jobs on every GPU; C5: a fixed job total split over the GPUs
    all_ranks = cfg["ranks"] * (1 if cfg.get("jobs_total") else world)
    all_lrs = cfg["lrs"] * (1 if cfg.get("jobs_total") else world)
    mine = PL.partition_jobs([per_job] * len(all_ranks), world)[rank]
    ranks_l, lrs_l = [all_ranks[j] for j in mine], [all_lrs[j] for j in mine]
    J = len(mine)
    rows = J * per_job
    seg = [j * per_job for j in range(J + 1)]

    # frozen base weights: created on rank 0, replicated once (NCCL broadcast over NVLink)
    W0 = {}
    for pi, (name, d, k, _) in enumerate(shapes):
        W0[name] = torch.empty(d, k, dtype=torch.bfloat16, device=dev)
        if rank == 0:  # U(-1, 1)/sqrt(k), the device's counter-based fill
            F.fill_uniform(W0[name], F.mix_seed(1234, 0, pi), -k ** -0.5, k ** -0.5)
    ctx = F.Context(dev)
    # one GPU per rank: the native communicator (libmlora.so -> NCCL), all W0 in one group
    comm, replication = None, "none (1 rank)" if world == 1 else "torch.distributed"
    if world > 1 and not share:
        try:
            comm, replication = PL.NativeComm(ctx), "mlora_broadcast_base (one NCCL group)"
        except Exception as e:  # setup only, never timed: keep the run alive, say so
            print(f"[bench] native communicator unavailable ({e}); W0 via torch.distributed", file=sys.stderr)
    comm_info = None
    if comm is not None:
        import ctypes
        from paper_2312_02515_b200 import _native as NL
        v = ctypes.c_int32()
        NL.lib().mlora_comm_nccl_version(ctypes.byref(v))
        comm_info = {"impl": "mlora_broadcast_base", "nranks": NL.lib().mlora_comm_size(comm.handle),
                     "nccl_version": v.value,
                     "bytes": sum(t.numel() * t.element_size() for t in W0.values())}
    t_bc = time.perf_counter()
    PL.broadcast_base_weights(W0, src=0, comm=comm)
    torch.cuda.synchronize()
    if comm_info is not None:
        comm_info["seconds"] = time.perf_counter() - t_bc
    if comm is not None:
        comm.close()  # the one-off replication is done: the steady state has no collective

    layer = FusedLoraLayer(ctx, shapes, ranks_l, [2.0] * J, lrs_l, rows, seed=1000 + rank, W0=W0)
    layer.set_layout(seg)
    xg = torch.Generator(device="cpu").manual_seed(77 + rank)
    x_host = (torch.rand(rows, shapes[0][2], generator=xg) * 2 - 1).to(torch.bfloat16).pin_memory()
    x = x_host.to(dev)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        return PL.max_over_ranks(v, device=dev)

    for _ in range(max(args.warmup, 3)):
        layer.step(x)
    barrier()

    # ---------------- device-resident timed region (headline `value`)
    sampler = ClockSampler(dev)
    launches0 = ctx.launches
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        layer.step(x)
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    launches = ctx.launches - launches0
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms_total / args.steps
    eff_tokens = int(PL.sum_over_ranks(rows, device=dev))  # δ = 0: every fused row is a real token
    value = eff_tokens * args.steps / (ms_total / 1e3)

    # ---------------- end-to-end (after the headline pass) through the public API with host buffers: every step's
    # 64 MiB hidden-state batch is copied H2D from pinned memory (copy stream, double
    # buffered so step i+1's upload overlaps step i) and its per-job losses D2H.
    from paper_2312_02515_b200.trainer import PipelinedTrainer
    trainer = PipelinedTrainer(layer, rows, shapes[0][2])
    losses_host = torch.empty(max(args.steps, 2), J, dtype=torch.float32).pin_memory()
    trainer.run([x_host] * 2, losses_host[:2])  # warm the pipeline
    barrier()
    time.sleep(1.5)  # the same rested-GPU regime as the headline pass (the power limiter relaxes)
    e2e_sampler = ClockSampler(dev)
    e2e_sampler.start()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    trainer.run([x_host] * args.steps, losses_host[:args.steps])
    f1.record(stream)
    barrier()
    e2e_clocks = e2e_sampler.stop()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1))
    e2e_value = eff_tokens * args.steps / (e2e_ms / 1e3)
    losses = losses_host[args.steps - 1].tolist()

    # ---------------- sustained: the same step for >= 1.2 s of device time, so the
    # board's power cap (1 kW, engaged within ~100 ms of load) and the capped SM
    # clock are in force and NVML has refreshed its readings several times
    sus_steps = max(args.steps, int(1200.0 / max(ms_step, 1e-3)) + 1)
    sus_sampler = ClockSampler(dev)
    sus_sampler.start()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    g0.record(stream)
    for _ in range(sus_steps):
        layer.step(x)
    g1.record(stream)
    barrier()
    sus_clocks = sus_sampler.stop()
    sus_ms = max_over_ranks(g0.elapsed_time(g1))
    sustained = {"value": eff_tokens * sus_steps / (sus_ms / 1e3), "unit": UNIT, "steps": sus_steps,
                 "ms_per_step": sus_ms / sus_steps, "clocks": sus_clocks}

    # ---------------- per-kernel live timing: the same K steps again with every launch
    # bracketed by CUDA events on its own stream (mlora_ctx_set_profiling).  Kept out of
    # the headline pass because events between launches defeat the PDL prologue overlap.
    # The board's power limiter needs ~1 s without load to lift the clock back to its
    # boost value; the pass then sees the same regime as the headline (a short burst
    # from a rested GPU) instead of the capped clock the sustained pass left behind.
    barrier()
    time.sleep(1.5)
    ctx.profile(reset=True)
    ctx.set_profiling(True)
    prof_sampler = ClockSampler(dev)
    prof_sampler.start()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        layer.step(x)
    p1.record(stream)
    barrier()
    prof_clocks = prof_sampler.stop()
    ctx.set_profiling(False)
    prof = ctx.profile(reset=True)
    prof_ms_total = p0.elapsed_time(p1)

    # ---------------- roofline of the dominant kernel (base GEMM, forward)
    peaks = load_peaks()
    cnt, ms = prof["base_fwd"]
    r_sum = sum(ranks_l)
    fl_fwd = sum(2 * rows * d * k + 2 * per_job * d * r_sum for _, d, k, _ in shapes)  # per step
    achieved = (fl_fwd * args.steps) / (ms / 1e3) / 1e12 if ms > 0 else None
    use_sustained = ms_total > 1000.0
    peak = peaks["bf16_sustained"] if use_sustained else peaks["bf16"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("base_fwd_dram_bytes_per_launch")
    fpt = flops_per_token(shapes, cfg["ranks"][0])
    step_tflops = value * fpt / 1e12
    kernel_share = {k: round(v[1] / max(sum(x[1] for x in prof.values()), 1e-9), 4) for k, v in prof.items()}
    kernel_ms_per_step = {k: round(v[1] / args.steps, 4) for k, v in prof.items()}

    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return 0

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            r = time_reference(cfg, steps=1, warmup=0)
            if r is not None:
                cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
                r1 = time_reference_single_core(cfg)
                if r1 is not None:
                    cpu["single_core"] = {k: r1[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # the baseline is reported, never the target
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if cfg.get("jobs_total") else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random tokens/weights, seeded)",
        "config": {"workload": cfg["workload"], "jobs_per_gpu": J, "ranks": cfg["ranks"], "lrs": cfg["lrs"],
                   "tokens_per_step_per_gpu": rows, "effective_tokens_per_step_per_gpu": rows,
                   "padding_ratio": 0.0, "parallelism": f"adapter-parallel (jobs partitioned) x{world}, "
                   f"W0 replicated once at init: {replication}",
                   "l2": "no flush; per-step working set (7 projections' W0 = 0.39 GB + activations) > 126 MB L2",
                   "flops_per_token": fpt},
        "step_tflops": step_tflops, "step_frac_of_peak": step_tflops / peak,
        "step_frac_of_sustained_peak": step_tflops / peaks["bf16_sustained"],
        "step_frac_of_burst_peak": step_tflops / peaks["bf16"],
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "frac_of_sustained": (achieved / peaks["bf16_sustained"]) if achieved else None,
                     "frac_of_burst": (achieved / peaks["bf16"]) if achieved else None,
                     "kernel": "mlora_base_pair_kernel (cta_group::2, 256x256 tile) forward: X W0^T + H B^T",
                     "peak_kind": ("sustained" if use_sustained else "burst") + " bf16, " + peaks["source"],
                     "launches": cnt, "avg_launch_us": 1e3 * ms / cnt if cnt else None,
                     "timed_in": "a separate pass of the same K steps after a 1.5 s rest, every launch bracketed "
                                 "by CUDA events on its stream", "clocks": prof_clocks},
        "kernel_time_share": kernel_share,
        "kernel_ms_per_step": kernel_ms_per_step,
        "profiled_pass_ms_per_step": prof_ms_total / args.steps,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": x_host.numel() * 2,
                "d2h_bytes_per_step": J * 4, "ms_per_step": e2e_ms / args.steps, "clocks": e2e_clocks},
        "sustained": sustained,
        "replication": comm_info,
        "gpu_launches": launches,
        "clocks": clocks,
        "losses": losses,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_decoder(args, cfg):
    """Model-level bench (--config c4): the whole decoder fine-tuning step per
    rank (jobs partitioned, frozen base broadcast once from rank 0, no
    steady-state collective), timed like the headline: CUDA events, max over ranks."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps({"impl": "reference", "unavailable": "the reference has no decoder / model arithmetic "
                              "(SURVEY.md App. A); its BatchFusion arm is --config c2"}))
        return 0
    import torch
    import torch.distributed as dist
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200 import model as MD
    from paper_2312_02515_b200 import parallel as PL

    share = os.environ.get("MLORA_BENCH_SHARE_GPU") == "1"  # multi-rank logic on a 1-GPU box (gloo)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if share:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    mc = MD.CONFIGS[cfg["decoder"]]
    if os.environ.get("MLORA_BENCH_LAYERS"):  # smaller smoke of the same path (never a reported number)
        mc = mc.with_layers(int(os.environ["MLORA_BENCH_LAYERS"]))
    per_job = cfg["seqs"] * cfg["seq_len"]
    all_ranks, all_lrs = cfg["ranks"] * world, cfg["lrs"] * world
    mine = PL.partition_jobs([per_job] * len(all_ranks), world)[rank]
    J = len(mine)
    g = torch.Generator().manual_seed(100 + rank)
    seqs = [[torch.randint(0, mc.vocab, (cfg["seq_len"],), generator=g).tolist() for _ in range(cfg["seqs"])]
            for _ in range(J)]
    batch = MD.pack_tokens(seqs)
    ctx = F.Context(dev)
    m = MD.MultiLoraDecoder(ctx, mc, [all_ranks[j] for j in mine], [2.0] * J, [all_lrs[j] for j in mine],
                            capacity=batch.rows, seed=1000 + rank)
    comm, replication = None, "none (1 rank)"
    if world > 1:
        if not share:
            try:
                comm, replication = PL.NativeComm(ctx), "mlora_broadcast_base (one NCCL group)"
            except Exception as e:
                replication = f"torch.distributed ({e})"
        else:
            replication = "torch.distributed (gloo, shared GPU)"
        PL.broadcast_base_weights(m.frozen_tensors(), src=0, comm=comm)
        torch.cuda.synchronize()
        if comm is not None:
            comm.close()  # the one-off replication is done: the steady state has no collective
    m.set_batch(batch)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        m.step()
    barrier()
    from paper_2312_02515_b200 import _native as NL
    sampler = ClockSampler(dev)
    launches0 = ctx.launches + NL.lib().mlora_free_launch_count()
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        m.step()
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    launches = ctx.launches + NL.lib().mlora_free_launch_count() - launches0
    ms_total = PL.max_over_ranks(e0.elapsed_time(e1), device=dev)
    eff = int(PL.sum_over_ranks(batch.real_tokens, device=dev))
    value = eff * args.steps / (ms_total / 1e3)
    # e2e through the public call with host token lists: set_batch (pinned H2D of
    # tokens / labels / mask / layout) + step + D2H of the per-job losses, every step
    host_loss = torch.empty(J, dtype=torch.float32).pin_memory()
    barrier()
    e2e_sampler = ClockSampler(dev)
    e2e_sampler.start()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        host_loss.copy_(m.step(batch), non_blocking=True)
    f1.record(stream)
    barrier()
    e2e_clocks = e2e_sampler.stop()
    e2e_ms = PL.max_over_ranks(f0.elapsed_time(f1), device=dev)
    # live per-kernel timing of the base GEMM (dominant kernel), a separate pass
    ctx.profile(reset=True)
    ctx.set_profiling(True)
    for _ in range(args.steps):
        m.step()
    barrier()
    ctx.set_profiling(False)
    prof = ctx.profile(reset=True)
    flops = m.flops_per_step()
    peaks = load_peaks()
    cnt, kms = prof["base_fwd"]
    lin_fwd = 0
    for li in range(mc.layers):
        for _, d, k in mc.projections():
            lin_fwd += 2 * batch.rows * d * k + 2 * batch.rows * d * cfg["ranks"][0]
    lin_fwd += 2 * batch.rows * mc.hidden * mc.vocab
    achieved = lin_fwd * args.steps / (kms / 1e3) / 1e12 if kms > 0 else None
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    line = {
        "metric": DECODER_METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random tokens/weights, seeded)",
        "config": {"workload": cfg["workload"].replace("28 layers", f"{mc.layers} layers"), "jobs_per_gpu": J,
                   "tokens_per_step_per_gpu": batch.rows,
                   "effective_tokens_per_step_per_gpu": batch.real_tokens,
                   "parallelism": f"adapter-parallel (jobs partitioned) x{world}, frozen base replicated once: "
                                  f"{replication}", "l2": "no flush; 12.5 GB of frozen weights per step >> L2",
                   "model_flops_per_step_per_gpu": flops},
        "step_tflops": flops * world / (ms_total / args.steps / 1e3) / 1e12,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16_sustained"], "unit": "TFLOP/s",
                     "frac": achieved / peaks["bf16_sustained"] if achieved else None, "traffic": None,
                     "frac_of_burst": achieved / peaks["bf16"] if achieved else None,
                     "kernel": "mlora_base_pair_kernel forward (every LoRA'd linear + the frozen LM head)",
                     "peak_kind": "sustained bf16, " + peaks["source"], "launches": cnt},
        "kernel_ms_per_step": {k: round(v[1] / args.steps, 3) for k, v in prof.items()},
        "e2e": {"value": eff * args.steps / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": 9 * batch.rows + 4 * (2 * len(batch.seq_lens) + 1 + J + 1),
                "d2h_bytes_per_step": 4 * J, "ms_per_step": e2e_ms / args.steps, "clocks": e2e_clocks},
        "gpu_launches": launches, "clocks": clocks, "losses": host_loss.tolist(),
        "cpu_baseline": None,
        "cpu_baseline_note": "the reference has no model arithmetic; its CPU path is per linear (--config c2)",
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
