"""The bench's batch leg (bench.batch_leg: batched prefill, ds_anchor_batch,
batched greedy decode) in isolation, with SM clocks sampled, so its anchor and
decode numbers can be compared with tools/anchor_alone.py --batch on one box:

    python tools/batch_leg_probe.py [--sizes 4,8]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2411_02820_b200 as P  # noqa: E402
from paper_2411_02820_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="4,8")
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--fragment-gb", type=float, default=0.0,
                help="allocate this much in 256 MB blocks and free every other one first (allocator state probe)")
args = ap.parse_args()
keep = []
if args.fragment_gb:
    blocks = [torch.empty(256 << 20, dtype=torch.uint8, device="cuda") for _ in range(int(args.fragment_gb * 4))]
    keep = blocks[::2]
    del blocks
n, k = args.n, 6
cfg = P.ModelConfig(max_seq=max(n, 8192) + 64, base_seed=0, mlp_kind="ungated", **dict(bench.SHAPE, vocab_size=128256))
L = cfg.n_layers
dev = torch.device("cuda", 0)
A = P.random_model(cfg, seed=1000, device=dev)
B = P.random_model(cfg, seed=2000, device=dev, base=A, perturb_layers=range(L - k, L), eps=0.5)
rc = P.RecomputeConfig([(L - k, L - 1)])
stream, side = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
sizes = [int(x) for x in args.sizes.split(",")]
with bench.ClockSampler(0) as clk:
    out = bench.batch_leg(P, _lib, cfg, A, B, rc, n, sizes, 1.0, 1.0, dev, stream, side)
clocks = clk.summary()
print(json.dumps({"sizes": {s: {k2: v[k2] for k2 in ("ttft_ms", "anchor_ms", "decode_ms_per_step")}
                            for s, v in out["sizes"].items()}, "clocks": clocks}))
