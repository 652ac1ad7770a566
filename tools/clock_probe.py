"""SM clock, power and throttle reasons while one workload's hta_forward runs back to back
(diagnostics).  usage: python tools/clock_probe.py [workload] [seconds]"""
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2502_17421_b200 import hta  # noqa: E402
from workloads.generators import config_workload  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "llama8b_64k"
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
    dev = torch.device("cuda:0")
    w = config_workload(name, seed=0)
    x = [t.to(dev) for t in (w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree)]
    mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
            time.sleep(0.02)

    for flush in (False, True):
        fl = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        hta.hta_forward(*x, mask)
        torch.cuda.synchronize()
        samples.clear()
        stop.clear()
        th = threading.Thread(target=sampler)
        th.start()
        t_end = time.time() + secs
        n = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        while time.time() < t_end:
            for _ in range(50):
                if flush:
                    fl.zero_()
                hta.hta_forward(*x, mask)
            n += 50
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        mhz = [s[0] for s in samples[len(samples) // 4:]]
        pw = [s[1] for s in samples[len(samples) // 4:]]
        reasons = sorted({s[2] for s in samples})
        print(f"{name} flush={flush}: {n} launches, {e0.elapsed_time(e1) / n * 1e3:.1f} us/launch; "
              f"SM MHz median {statistics.median(mhz):.0f} min {min(mhz)} max {max(mhz)}; "
              f"power median {statistics.median(pw):.0f} W max {max(pw):.0f}; reasons {[hex(r) for r in reasons]}")


if __name__ == "__main__":
    main()
