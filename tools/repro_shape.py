"""Debug: a forced-persistent 8K partial prefill, then a 16K full prefill
(the sequence the crossover sweep runs), eager, synchronising after each call."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402

SHAPE = dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab_size=128256)
steps = [(8192, 3), (16384, 32)]
if len(sys.argv) > 1:
    steps = [tuple(int(x) for x in s.split(":")) for s in sys.argv[1:]]
for n, k in steps:
    cfg = P.ModelConfig(max_seq=n + 64, base_seed=0, **SHAPE)
    L = 32
    A = P.random_model(cfg, seed=1)
    B = P.random_model(cfg, seed=2, base=A, perturb_layers=range(L - k, L)) if k < L else A
    ids = np.random.default_rng(3).integers(0, cfg.vocab_size, size=n, dtype=np.int64)
    tok = torch.from_numpy(ids).cuda()
    side = torch.cuda.Stream()
    if k == L:
        r = P.full_prefill(B, ids, e_layers=(), copy_stream=side, tokens_dev=tok)
    else:
        rc = P.RecomputeConfig([(L - k, L - 1)])
        prod = P.full_prefill(A, ids, e_layers=rc.transition_layers, tokens_dev=tok)
        torch.cuda.synchronize()
        print("producer ok", n, flush=True)
        r = P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), copy_stream=side, tokens_dev=tok)
    torch.cuda.synchronize()
    print("ok", n, k, float(r.logits.float().abs().sum()), flush=True)
    del A, B
    torch.cuda.empty_cache()
