"""How fast do NVML's SM clock, clock-event reasons and instantaneous power move?
Samples them every 1 ms from a side thread while bf16 GEMMs run for a few
seconds. Prints each change with its timestamp. bench.py's clock evidence comes
from these same calls."""
import threading
import time

import pynvml as nv
import torch


def main():
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    fi = nv.NVML_FI_DEV_POWER_INSTANT
    log, halt = [], threading.Event()

    def sample():
        t0 = time.perf_counter()
        while not halt.is_set():
            clk = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            fv = nv.nvmlDeviceGetFieldValues(h, [fi])[0]
            pw = fv.value.uiVal / 1000 if fv.nvmlReturn == 0 else -1
            log.append((time.perf_counter() - t0, clk, rs, pw, nv.nvmlDeviceGetPowerUsage(h) / 1000))
            time.sleep(0.001)

    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    th = threading.Thread(target=sample, daemon=True)
    th.start()
    time.sleep(0.3)  # idle baseline
    ev = []
    for i in range(300):  # ~1.1 TFLOP each: about 3 s of GEMMs
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        torch.mm(a, b)
        ev.append(e)
    end = torch.cuda.Event(enable_timing=True)
    end.record()
    torch.cuda.synchronize()
    time.sleep(0.5)
    halt.set()
    th.join()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(ev) - 1)] + [ev[-1].elapsed_time(end)]
    print("gemm ms: first10", [round(x, 3) for x in ms[:10]], "last10", [round(x, 3) for x in ms[-10:]])
    last = None
    for t, clk, rs, pw, pavg in log:
        key = (clk, rs, pw)
        if key != last:
            print(f"t={t:7.3f}s clk={clk} reasons=0x{rs:x} p_inst={pw:.0f}W p_avg={pavg:.0f}W")
            last = key
    print("samples", len(log))


if __name__ == "__main__":
    main()
