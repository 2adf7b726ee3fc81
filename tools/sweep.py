"""BASELINE config 5: prefix-length x recompute-fraction sweep on one B200.

n in {2K, 4K, 8K, 16K, 32K} x k in {3, 6, 10, 13, 16} of 32 layers recomputed
(suffix group [32-k, 31], the profiler-consistent set for B = A + noise on
that suffix).  For each point: consumer TTFT (partial prefill,
CUDA graph, CUDA events, median) vs the same GPU's full prefill.

    python tools/sweep.py [--ns 2048,4096,...] [--ks 3,6,...] [--steps 5] > profiles/r01_sweep.json
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402

SHAPE = dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab_size=128256)


def timed(fn, steps, stream):
    ts = []
    for _ in range(steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        with torch.cuda.stream(stream):
            fn()
        e.record(stream)
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="2048,4096,8192,16384,32768")
    ap.add_argument("--ks", default="3,6,10,13,16")
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    ns = [int(x) for x in args.ns.split(",")]
    ks = [int(x) for x in args.ks.split(",")]
    cfg = P.ModelConfig(max_seq=max(ns), base_seed=0, **SHAPE)
    L = cfg.n_layers
    A = P.random_model(cfg, seed=1000)
    B = P.random_model(cfg, seed=2000, base=A, perturb_layers=range(L - max(ks), L), eps=0.5)
    stream, side = torch.cuda.Stream(), torch.cuda.Stream()
    rows = []
    for n in ns:
        ids = np.random.default_rng(n).integers(0, cfg.vocab_size, size=n, dtype=np.int64)
        tok = torch.from_numpy(ids).cuda()
        prod = P.full_prefill(A, ids, e_layers=[L - k for k in ks], tokens_dev=tok)
        torch.cuda.synchronize()  # the producer ran on the default stream: finish it before timing
        full = timed(lambda: P.full_prefill(B, ids, e_layers=(), stream=stream, copy_stream=side, tokens_dev=tok), 1 + args.steps,
                     stream)
        cache = P.PagedKV.allocate(cfg, n)
        for k in ks:
            rc = P.RecomputeConfig([(L - k, L - 1)])

            def step():
                return P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, stream=stream,
                                         copy_stream=side, tokens_dev=tok)

            with torch.cuda.stream(stream):
                step()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step()
            for _ in range(2):
                with torch.cuda.stream(stream):
                    g.replay()
            ttft = timed(g.replay, args.steps, stream)
            rows.append({"n": n, "k": k, "frac": k / L, "ttft_ms": round(ttft, 3), "full_ms": round(full, 3),
                         "speedup": round(full / ttft, 3), "tok_s": round(n / ttft * 1e3, 1)})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            del g
        del prod, cache
        torch.cuda.empty_cache()
    print(json.dumps({"sweep": rows, "shape": "Llama-3-8B-shaped ref block (ungated MLP), bf16",
                      "device": torch.cuda.get_device_name()}))


if __name__ == "__main__":
    main()
