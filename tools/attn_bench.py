"""Time the prefill attention kernel alone at the 8B shape (CUDA events).

    python tools/attn_bench.py [--n 8192]        (DS_FA_LEGACY=1 for the mma.sync kernel)
"""
import argparse
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_02820_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
args = ap.parse_args()
H, G, D = 32, 8, 128
P = args.n - 1
pages = (args.n + 63) // 64
kc = torch.randn(1, pages, G, 64, D, device="cuda").bfloat16()
vc = torch.randn(1, pages, G, 64, D, device="cuda").bfloat16()
table = torch.arange(pages, dtype=torch.int32, device="cuda")
q = torch.randn(P, H * D, device="cuda").bfloat16()
o = torch.empty_like(q)
desc = ops.paged_kv_desc(kc, vc, table, args.n)
for _ in range(3):
    ops.attention_prefill(q, desc, 0, H, G, D, out=o)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    ops.attention_prefill(q, desc, 0, H, G, D, out=o)
    e.record()
    e.synchronize()
    ts.append(s.elapsed_time(e))
ms = statistics.median(ts)
flops = 4 * H * D * P * (P + 1) / 2
print(f"attention n={args.n}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s (causal pairs)")
