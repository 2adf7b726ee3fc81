"""Sustained GEMM throughput at the power cap: our CTA-pair tcgen05 GEMM vs
cuBLAS (torch.matmul) on the recompute's W1 shape (M=8191, N=14336, K=4096),
each looped for a few seconds while NVML samples clocks and power.

    python tools/gemm_cap.py [--secs 3]
"""
import argparse
import math
import statistics
import sys
import threading
import time
from pathlib import Path

import pynvml
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_02820_b200 import _lib as L, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--secs", type=float, default=3.0)
args = ap.parse_args()
M, N, K = 8191, 14336, 4096
a = torch.randn(M, K, device="cuda").bfloat16()
w = (torch.randn(N, K, device="cuda") / math.sqrt(K)).bfloat16()
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
wt = w.t()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
cases = {
    "ours_store": lambda: ops.gemm(a, w, mode=L.EPI_STORE_BF16, out=out),
    "ours_silu": lambda: ops.gemm(a, w, mode=L.EPI_SILU_BF16, out=out),
    "cublas": lambda: torch.matmul(a, wt, out=out),
}
for name, fn in cases.items():
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.02)

    th = threading.Thread(target=sampler)
    th.start()
    ts, t_end = [], time.time() + args.secs
    while time.time() < t_end:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 10)
    stop.set()
    th.join()
    late = samples[len(samples) // 3:]
    ms = statistics.median(ts[len(ts) // 3:])
    print(f"{name:11s} {ms:.4f} ms  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s  sm_mhz {statistics.median(x[0] for x in late):5.0f}"
          f"  power_w {statistics.median(x[1] for x in late):5.0f}")
    time.sleep(1.0)
