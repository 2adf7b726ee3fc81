"""Consumer step time at BASELINE config 2 (n = 8192, k = 6, two streams, CUDA
graph), median of --steps after --warmup; for same-box A/B via tools/ab_run.py.

    python tools/step_time.py [--n 8192] [--k 6] [--steps 30]
"""
import argparse
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--k", type=int, default=6)
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--warmup", type=int, default=10)
args = ap.parse_args()
SHAPE = dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab_size=128256)
cfg = P.ModelConfig(max_seq=args.n + 64, base_seed=0, **SHAPE)
L, k, n = 32, args.k, args.n
A = P.random_model(cfg, seed=1000)
B = P.random_model(cfg, seed=2000, base=A, perturb_layers=range(L - k, L), eps=0.5)
rc = P.RecomputeConfig([(L - k, L - 1)])
ids = np.random.default_rng(7).integers(0, cfg.vocab_size, size=n, dtype=np.int64)
tok = torch.from_numpy(ids).cuda()
prod = P.full_prefill(A, ids, e_layers=rc.transition_layers, tokens_dev=tok)
torch.cuda.synchronize()
cap = P.CapturedPartialPrefill(B, n, rc, prod.kv, prod.e_map())
s = cap.stream
ts = []
for i in range(args.warmup + args.steps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    with torch.cuda.stream(s):
        cap.graph.replay()
    b.record(s)
    torch.cuda.synchronize()
    if i >= args.warmup:
        ts.append(a.elapsed_time(b))
print(f"step n={n} k={k}: p50 {statistics.median(ts):.3f} ms  min {min(ts):.3f}  max {max(ts):.3f}")
