"""One consumer partial-prefill step at BASELINE config 2 for ncu.

The producer export and warm-up run outside the profiled range; only the
consumer step sits between cudaProfilerStart/Stop, so run ncu with
``--profile-from-start off``:

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python tools/profile_step.py
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--k", type=int, default=6)
ap.add_argument("--what", default="partial", choices=["partial", "full"])
ap.add_argument("--single", action="store_true", help="one stream (per-launch anchor kernels)")
args = ap.parse_args()

cfg = P.ModelConfig(32, 4096, 32, 8, 128, 14336, 128256, max(args.n, 8192), 0)
L = cfg.n_layers
A = P.random_model(cfg, seed=1000)
B = P.random_model(cfg, seed=2000, base=A, perturb_layers=range(L - args.k, L))
rc = P.RecomputeConfig([(L - args.k, L - 1)])
ids = np.random.default_rng(7).integers(0, cfg.vocab_size, size=args.n, dtype=np.int64)
tok = torch.from_numpy(ids).cuda()
prod = P.full_prefill(A, ids, e_layers=rc.transition_layers, tokens_dev=tok)
cache = P.PagedKV.allocate(cfg, args.n)
side = None if args.single else torch.cuda.Stream()
for _ in range(2):
    P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, copy_stream=side, tokens_dev=tok)
torch.cuda.synchronize()
torch.cuda.profiler.start()
if args.what == "partial":
    P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, copy_stream=side, tokens_dev=tok)
else:
    P.full_prefill(B, ids, e_layers=(), tokens_dev=tok)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
