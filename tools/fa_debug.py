"""Per-(head, 128-row tile) error map of the prefill attention against fp32 torch."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_02820_b200 import ops  # noqa: E402

n, H, G, D = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (1000, 8, 2, 128)))
g = torch.Generator(device="cuda").manual_seed(n + H)
k = torch.randn(1, G, n, D, device="cuda", generator=g).bfloat16()
v = torch.randn(1, G, n, D, device="cuda", generator=g).bfloat16()
q = torch.randn(n, H * D, device="cuda", generator=g).bfloat16()
out = ops.attention_prefill(q, ops.dense_kv_desc(k, v), 0, H, G, D).float()
R = H // G
qh = q.float().view(n, H, D).transpose(0, 1)
kk = k[0].float().repeat_interleave(R, 0)
vv = v[0].float().repeat_interleave(R, 0)
s = qh @ kk.transpose(1, 2) / math.sqrt(D)
mask = torch.arange(n, device="cuda")[None, :] > torch.arange(n, device="cuda")[:, None]
s = s.masked_fill(mask, float("-inf"))
ref = (torch.softmax(s, -1) @ vv).transpose(0, 1).reshape(n, H * D)
err = (out - ref).abs().view(n, H, D).amax(-1)  # [n, H]
for h in range(H):
    row = []
    for t in range(0, n, 128):
        row.append(f"{err[t:t + 128, h].max().item():.2f}")
    print(f"head {h}: " + " ".join(row))
bad = (err > 0.05).nonzero()
print("bad rows (first 20):", bad[:20].tolist())
