"""Clock / power under each workload of the consumer step (BASELINE config 2):
recompute alone, anchor alone, the fused two-stream step, the single-stream step.
Each runs back to back as CUDA-graph replays for ~3 s while a thread samples
NVML (SM clock, power, throttle reasons); prints ms per replay and medians.

    python tools/power_probe.py [--n 8192] [--k 6] [--secs 3]
"""
import argparse
import ctypes as C
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np
import pynvml
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402
from paper_2411_02820_b200 import _lib as L  # noqa: E402
from paper_2411_02820_b200.engine import _workspace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--k", type=int, default=6)
ap.add_argument("--secs", type=float, default=3.0)
args = ap.parse_args()
cfg = P.ModelConfig(32, 4096, 32, 8, 128, 14336, 128256, max(args.n, 8192), 0)
Lh, n, k = cfg.n_layers, args.n, args.k
A = P.random_model(cfg, seed=1000)
B = P.random_model(cfg, seed=2000, base=A, perturb_layers=range(Lh - k, Lh))
rc = P.RecomputeConfig([(Lh - k, Lh - 1)])
ids = np.random.default_rng(7).integers(0, cfg.vocab_size, size=n, dtype=np.int64)
tok = torch.from_numpy(ids).cuda()
prod = P.full_prefill(A, ids, e_layers=rc.transition_layers, tokens_dev=tok)
cache = P.PagedKV.allocate(cfg, n)
s, side = torch.cuda.Stream(), torch.cuda.Stream()
ws = _workspace(B, n, s)
lib = L.lib()
e = prod.e_map()[Lh - k].hidden
d = cache.desc()
logits = torch.empty(cfg.vocab_size, device="cuda")
t32 = torch.empty(1, dtype=torch.int32, device="cuda")


def recompute():
    L.check(lib.ds_recompute_group(C.byref(B.desc()), tok.data_ptr(), n, Lh - k, Lh - 1, e.data_ptr(), e.shape[0],
                                   C.byref(d), ws.data_ptr(), ws.numel(), s.cuda_stream))


def anchor():
    L.check(lib.ds_anchor(C.byref(B.desc()), tok.data_ptr(), n, C.byref(d), logits.data_ptr(), t32.data_ptr(),
                          ws.data_ptr(), ws.numel(), s.cuda_stream))


work = {
    "recompute": recompute,
    "anchor": anchor,
    "two_stream": lambda: P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, stream=s, copy_stream=side,
                                            tokens_dev=tok),
    "single_stream": lambda: P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, stream=s, tokens_dev=tok),
}
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
for name, fn in work.items():
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
            time.sleep(0.02)

    th = threading.Thread(target=sampler)
    th.start()
    ts, t_end = [], time.time() + args.secs
    while time.time() < t_end:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        with torch.cuda.stream(s):
            g.replay()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    stop.set()
    th.join()
    late = samples[len(samples) // 3:]
    print(f"{name:14s} replays {len(ts):4d}  ms p50 {statistics.median(ts):7.3f} (first {ts[0]:.3f}, last {ts[-1]:.3f})"
          f"  sm_mhz p50 {statistics.median(x[0] for x in late):6.0f}  power_w p50 {statistics.median(x[1] for x in late):6.0f}"
          f"  reasons {sorted(set(x[2] for x in late))}")
    time.sleep(1.0)
