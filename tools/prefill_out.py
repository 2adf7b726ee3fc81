"""Save a producer full prefill and a consumer partial prefill (logits + KV) of a
seeded model, for bitwise comparisons between build switches read once per
process (e.g. DS_GEMM_EPI_WARPS, DS_FA_VARIANT).

    DS_GEMM_EPI_WARPS=8 python tools/prefill_out.py --out /tmp/a.pt
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4095)
ap.add_argument("--out", required=True)
args = ap.parse_args()
cfg = P.ModelConfig(n_layers=6, d_model=2048, n_heads=16, n_kv_heads=4, head_dim=128, d_ff=5632, vocab_size=8192,
                    max_seq=args.n + 64, base_seed=0)
A = P.random_model(cfg, seed=5)
B = P.random_model(cfg, seed=6, base=A, perturb_layers=range(3, 6), eps=0.5)
ids = np.random.default_rng(9).integers(0, cfg.vocab_size, size=args.n, dtype=np.int64)
rc = P.RecomputeConfig([(3, 5)])
prod = P.full_prefill(A, ids, e_layers=rc.transition_layers)
cons = P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), copy_stream=torch.cuda.Stream())
torch.cuda.synchronize()
cd = cons.kv.dense()
torch.save({"prod_logits": prod.logits.cpu(), "prod_k": prod.kv.k.cpu(), "cons_logits": cons.logits.cpu(),
            "cons_k": cd.k.cpu(), "cons_v": cd.v.cpu(), "token": cons.token}, args.out)
print("saved", args.out, bool(torch.isfinite(cons.logits).all()))
