"""A fused consumer call (persistent co-resident anchor) while another
stream's work -- a producer prefill on the default stream, with its per-launch
anchor kernels -- is still running on the same GPU.  Every stand-alone kernel
must fit beside one anchor CTA per SM, or the fused call can starve.

    python tools/concurrency_check.py [--n 16384] [--reps 3]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
SHAPE = dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab_size=128256)
cfg = P.ModelConfig(max_seq=args.n, base_seed=0, **SHAPE)
A = P.random_model(cfg, seed=1)
B = P.random_model(cfg, seed=2, base=A, perturb_layers=range(29, 32))
ids = np.random.default_rng(3).integers(0, cfg.vocab_size, size=args.n, dtype=np.int64)
tok = torch.from_numpy(ids).cuda()
s, side = torch.cuda.Stream(), torch.cuda.Stream()
ref = P.full_prefill(B, ids, e_layers=(), stream=s, copy_stream=side, tokens_dev=tok)
torch.cuda.synchronize()
want = ref.logits.clone()
for r in range(args.reps):
    P.full_prefill(A, ids, e_layers=(29,), tokens_dev=tok)  # default stream, not synchronised
    got = P.full_prefill(B, ids, e_layers=(), stream=s, copy_stream=side, tokens_dev=tok)
    torch.cuda.synchronize()
    assert torch.equal(got.logits, want), "results differ under concurrency"
    print("rep", r, "ok", flush=True)
print("concurrency ok")
