"""Small batched prefill + batched decode + dual FA for compute-sanitizer (TINY and a d=2048 shape)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402
from paper_2411_02820_b200.quality import decode_greedy_batch  # noqa: E402

for dims in (dict(n_layers=4, d_model=256, n_heads=4, n_kv_heads=1, head_dim=64, d_ff=1024, vocab_size=4096,
                  max_seq=1024, base_seed=7),
             dict(n_layers=2, d_model=2048, n_heads=16, n_kv_heads=4, head_dim=128, d_ff=4096, vocab_size=8192,
                  max_seq=1024, base_seed=5)):
    cfg = P.ModelConfig(**dims)
    A = P.random_model(cfg, seed=1)
    B = P.random_model(cfg, seed=2, base=A, perturb_layers=range(cfg.n_layers - 1, cfg.n_layers), eps=0.5)
    rng = np.random.default_rng(0)
    toks = [rng.integers(0, cfg.vocab_size, size=n, dtype=np.int64) for n in (200, 131, 64)]
    rc = P.RecomputeConfig([(cfg.n_layers - 1, cfg.n_layers - 1)])
    prods = [P.full_prefill(A, t, e_layers=rc.transition_layers) for t in toks]
    outs = P.partial_prefill_batch(B, toks, rc, [p.kv for p in prods], [p.e_map() for p in prods],
                                   out=[P.PagedKV.allocate(cfg, len(t) + 4) for t in toks],
                                   copy_stream=torch.cuda.Stream())
    decode_greedy_batch(B, [o.kv for o in outs], outs, 4, [len(t) for t in toks])
    torch.cuda.synchronize()
    print("ok", dims["d_model"])
