"""Where a batched decode's caches differ from per-sequence decodes (debug)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402
from paper_2411_02820_b200.quality import decode_greedy, decode_greedy_batch  # noqa: E402

cfg = P.ModelConfig(n_layers=3, d_model=2048, n_heads=16, n_kv_heads=4, head_dim=128, d_ff=4096, vocab_size=16384,
                    max_seq=2048, base_seed=5)
A = P.random_model(cfg, seed=11)
LENGTHS = [300, 257, 512, 129, 64, 700, 2, 411]
for nb in (2, 4, 5):
    rng = np.random.default_rng(5)
    steps = 12
    toks = [rng.integers(0, cfg.vocab_size, size=LENGTHS[b] + 3, dtype=np.int64) for b in range(nb)]
    caches, lasts = [], []
    for t in toks:
        kv = P.LayerKV.empty(cfg, len(t) + steps)
        lasts.append(P.full_prefill(A, t, e_layers=[], out=kv))
        caches.append(kv)
    copies = [P.LayerKV(c.k.clone(), c.v.clone()) for c in caches]
    one = [decode_greedy(A, c, last, steps, positions=len(t)) for c, last, t in zip(copies, lasts, toks)]
    got = decode_greedy_batch(A, caches, lasts, steps, [len(t) for t in toks])
    for b in range(nb):
        for name in ("k", "v"):
            x, y = getattr(caches[b], name), getattr(copies[b], name)
            bad = (x != y).nonzero()
            if len(bad):
                pos = sorted(set(bad[:, 2].tolist()))
                layers = sorted(set(bad[:, 0].tolist()))
                heads = sorted(set(bad[:, 1].tolist()))
                print(f"nb={nb} row {b} ({len(toks[b])} tok) {name}: {len(bad)} diffs, layers {layers}, heads {heads}, "
                      f"positions {pos[:8]}..{pos[-3:]}, maxdiff {float((x.float() - y.float()).abs().max()):.3g}",
                      flush=True)
        print(f"nb={nb} row {b}: tokens equal {np.array_equal(got[b], one[b])}", flush=True)
