"""§8f row 3 on the device: the product's measured memory model drives the
executor's admission.

Live warm-up probes (memory.probe_samples: the warmup_plan cross product, each
probe one real fused LLaMA-7B-layer step read through cudaMemGetInfo) are fitted
by the product's fit_memory_model and agree with the reference's own fit of the
same samples.  Then FusedExecutor runs 6 jobs under a budget smaller than all of
them: every iteration it fuses exactly the jobs the reference's schedule()
(scheduler.cpp:74-130, compiled in place) admits from the same queue state, and
the measured footprint of every admitted set (the same cudaMemGetInfo probe, its
jobs and rows) stays under the budget."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ref  # noqa: E402

pytestmark = pytest.mark.gpu


def ref_schedule(L, queue, strategy, beta, budget, floor, M):
    n = len(queue)
    L.ref_schedule.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_int), C.POINTER(C.c_double),
                               C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_long),
                               C.POINTER(C.c_double), C.c_int, C.c_int, C.POINTER(C.c_double), C.c_double,
                               C.c_double, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double)]
    flat = [x for q in queue for x in q["lengths"]]
    out, cnt, est = (C.c_int * n)(), C.c_int(), C.c_double()
    rc = L.ref_schedule(n, (C.c_char_p * n)(*[q["id"].encode() for q in queue]),
                        (C.c_int * n)(*[q["priority"] for q in queue]),
                        (C.c_double * n)(*[q["submit"] for q in queue]), (C.c_int * n)(*[q["bs"] for q in queue]),
                        (C.c_int * n)(*[len(q["lengths"]) for q in queue]), (C.c_int * len(flat))(*flat),
                        (C.c_long * n)(*[q["cursor"] for q in queue]), (C.c_double * n)(*([0.0] * n)),
                        {"fifo": 0, "priority": 1, "minpad": 2}[strategy], 1, (C.c_double * 3)(*beta), budget, floor,
                        M, out, C.byref(cnt), C.byref(est))
    assert rc == 0
    return [out[i] for i in range(cnt.value)], est.value


@pytest.mark.parametrize("strategy", ["minpad", "fifo"])
def test_executor_admits_under_measured_memory_model(strategy):
    from paper_2312_02515_b200 import fused as F
    from paper_2312_02515_b200 import memory as MM
    from paper_2312_02515_b200 import packer as P
    from paper_2312_02515_b200.executor import FusedExecutor, JobConfig
    from paper_2312_02515_b200.layer import LLAMA7B
    if not ref.available() and not ref.build():
        pytest.skip("reference checker unavailable")
    L = ref.lib()
    dev = torch.device("cuda", 0)
    W0 = {}
    for pi, (name, d, k, _) in enumerate(LLAMA7B):
        W0[name] = F.fill_uniform(torch.empty(d, k, dtype=torch.bfloat16, device=dev), F.mix_seed(9, 0, pi),
                                  -k ** -0.5, k ** -0.5)
    # ---- warm-up: live probes -> the product's fit == the reference's fit of the same samples
    samples = MM.probe_samples(dev, LLAMA7B, 16, [1, 2, 4], [128, 256, 512], W0)
    model = MM.fit_memory_model(samples)
    n = len(samples)
    out = (C.c_double * 4)()
    L.ref_fit_memory_model.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                       C.c_int, C.POINTER(C.c_double)]
    assert L.ref_fit_memory_model(n, (C.c_int * n)(*[s[0] for s in samples]), (C.c_int * n)(*[s[1] for s in samples]),
                                  (C.c_double * n)(*[s[2] for s in samples]), 0, out) == 0
    assert np.allclose([model.beta0, model.beta1, model.beta2], list(out)[:3], rtol=1e-6, atol=1e-12)
    print("memory probes (batch_size, seq_len, GB):", [(b, l, round(m, 4)) for b, l, m in samples])
    assert model.beta1 > 0 and model.rmse < 0.01, (model, samples)
    # ---- 6 jobs under a budget that holds about half of them
    jobs = []
    for j in range(6):
        lengths = P.sample_lengths("uniform", 6, seed=300 + j, min_len=64, max_len=128 * (1 + j % 4))
        jobs.append(JobConfig(f"job{j}", lengths, batch_size=1 + j % 3, rank=16, lr=1e-4, priority=1 + j % 2,
                              submit_time=float(j % 3), iterations=3))
    floor = 0.1
    est = [model.predict_clamped(jc.batch_size, max(jc.lengths), floor) for jc in jobs]
    budget = 0.5 * sum(est)
    ctx = F.Context(dev)
    ex = FusedExecutor(ctx, LLAMA7B, jobs, max_concurrent=4, strategy=strategy, seed=3, W0=W0, pipelined=False,
                       memory_budget_gb=budget, memory_model=model, memory_floor_gb=floor)
    measured = {}
    steps = 0
    while ex.active() and not ex.trace.truncated:
        live = ex.active()
        queue = [dict(id=ex.jobs[i].cfg.id, priority=ex.jobs[i].cfg.priority, submit=ex.jobs[i].cfg.submit_time,
                      bs=ex.jobs[i].cfg.batch_size, lengths=list(ex.jobs[i].cfg.lengths), cursor=ex.jobs[i].cursor)
                 for i in live]
        want, want_gb = ref_schedule(L, queue, strategy, [model.beta0, model.beta1, model.beta2], budget, floor, 4)
        ev = ex.step()
        steps += 1
        assert ev["routing"] == [queue[q]["id"] for q in want]
        assert ev["estimated_memory_gb"] == pytest.approx(want_gb)
        assert ev["estimated_memory_gb"] <= budget + 1e-9
        key = (tuple(sorted(ev["routing"])), ev["rows"])
        if key not in measured:
            measured[key] = MM.measure_step_gb(dev, LLAMA7B, [16] * len(key[0]), ev["rows"], W0)
            assert measured[key] <= budget, (key, measured[key], budget)
            assert measured[key] <= ev["estimated_memory_gb"] * 1.05, (key, measured[key], ev)
    assert steps > 0 and not ex.trace.truncated
    print(f"{strategy}: {steps} iterations under {budget:.3f} GB; model b0={model.beta0:.4f} GB "
          f"b1={model.beta1 * 1e6:.1f} KB/token; measured admitted sets: "
          f"{ {k: round(v, 3) for k, v in measured.items()} }")
