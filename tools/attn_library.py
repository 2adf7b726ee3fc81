"""Prefill attention at the 8B shape: our tcgen05 kernel vs the Blackwell
library kernels on the same box (SURVEY §7.3 / VERDICT r1: a Blackwell-native
library attention baseline).

    python tools/attn_library.py [--n 8192] [--reps 20] [--out profiles/r02_attention_library.json]

Shape: one layer of the Llama-3-8B-shaped block, H 32 / KVH 8 / D 128, causal
over the n-1 window.  FLOPs = 4 * H * D * P(P+1)/2 (causal pairs only) for
every row.  Each implementation is timed with CUDA events on the current
stream (median of --reps after 3 warm-ups) and its output is compared with
ours (rel-L2).  Libraries: torch SDPA on the cuDNN backend, flashinfer's
CuTe-DSL Blackwell FMHA (BatchPrefillCuteDSLWrapper, FA4-style warp-specialised
tcgen05 kernel, JIT-compiled in process), flash_attn 2.8 (sm80-class).
"""
import argparse
import json
import math
import statistics
import sys
import traceback
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2411_02820_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--out", default="")
args = ap.parse_args()
H, G, D = 32, 8, 128
P = args.n - 1
flops = 4 * H * D * P * (P + 1) / 2
torch.manual_seed(0)
q = torch.randn(P, H, D, device="cuda").bfloat16()
k = torch.randn(P, G, D, device="cuda").bfloat16()
v = torch.randn(P, G, D, device="cuda").bfloat16()
scale = 1.0 / math.sqrt(D)


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


rows = []

# ---- ours: paged cache [1, pages, G, 64, D]
pages = (args.n + 63) // 64
kc = torch.zeros(1, pages, G, 64, D, device="cuda", dtype=torch.bfloat16)
vc = torch.zeros_like(kc)
kc.view(1, -1, 64, D)  # noqa
for p in range(pages):
    lo, hi = p * 64, min(P, p * 64 + 64)
    if lo < hi:
        kc[0, p, :, :hi - lo] = k[lo:hi].transpose(0, 1)
        vc[0, p, :, :hi - lo] = v[lo:hi].transpose(0, 1)
table = torch.arange(pages, dtype=torch.int32, device="cuda")
desc = ops.paged_kv_desc(kc, vc, table, args.n)
q2 = q.reshape(P, H * D)
o_ours = torch.empty_like(q2)
ms = timeit(lambda: ops.attention_prefill(q2, desc, 0, H, G, D, out=o_ours))
ref = o_ours.float().view(P, H, D)
rows.append({"impl": "ours fa_tc_kernel (tcgen05/TMEM, paged KV)", "ms": ms, "tflops": flops / ms / 1e9})


def add(name, fn, get):
    try:
        ms = timeit(fn)
        out = get().float().reshape(P, H, D)
        rel = float((out - ref).norm() / ref.norm())
        rows.append({"impl": name, "ms": ms, "tflops": flops / ms / 1e9, "rel_l2_vs_ours": rel})
    except Exception as exc:  # report, keep going
        rows.append({"impl": name, "unavailable": f"{type(exc).__name__}: {exc}"[:300]})
        traceback.print_exc()


# ---- torch SDPA, cuDNN backend ([B, H, S, D]; GQA expanded to H heads for the backends without it)
try:
    from torch.nn.attention import SDPBackend, sdpa_kernel
    qt = q.transpose(0, 1).unsqueeze(0)
    ke = k.repeat_interleave(H // G, 1).transpose(0, 1).unsqueeze(0).contiguous()
    ve = v.repeat_interleave(H // G, 1).transpose(0, 1).unsqueeze(0).contiguous()
    box = {}

    def cudnn():
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            box["o"] = torch.nn.functional.scaled_dot_product_attention(qt, ke, ve, is_causal=True, scale=scale)

    add("torch SDPA cuDNN backend (GQA expanded)", cudnn, lambda: box["o"][0].transpose(0, 1))

    def flash_sdpa():
        with sdpa_kernel([SDPBackend.FLASH_ATTENTION]):
            box["f"] = torch.nn.functional.scaled_dot_product_attention(qt, ke, ve, is_causal=True, scale=scale)

    add("torch SDPA flash backend (GQA expanded)", flash_sdpa, lambda: box["f"][0].transpose(0, 1))
except Exception as exc:
    rows.append({"impl": "torch SDPA", "unavailable": str(exc)[:300]})

# ---- flashinfer CuTe-DSL Blackwell FMHA (FA4-style)
try:
    from flashinfer.cute_dsl.attention.wrappers.batch_prefill import BatchPrefillCuteDSLWrapper
    ws = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
    w = BatchPrefillCuteDSLWrapper(ws)
    ind = torch.tensor([0, P], dtype=torch.int32, device="cuda")
    w.plan(ind, ind, H, G, D, causal=True, sm_scale=scale, q_data_type=torch.bfloat16,
           kv_data_type=torch.bfloat16)
    box2 = {}

    def fi():
        box2["o"] = w.run(q, k, v)

    add("flashinfer CuTe-DSL sm100 FMHA (BatchPrefillCuteDSLWrapper)", fi, lambda: box2["o"])
except Exception as exc:
    rows.append({"impl": "flashinfer CuTe-DSL sm100 FMHA", "unavailable": f"{type(exc).__name__}: {exc}"[:300]})
    traceback.print_exc()

# ---- flash_attn 2.8 (sm80-class kernels on B200)
try:
    from flash_attn import flash_attn_func
    qf, kf, vf = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)
    box3 = {}

    def fa2():
        box3["o"] = flash_attn_func(qf, kf, vf, causal=True, softmax_scale=scale)

    add("flash_attn 2.8.3 (sm80 kernels)", fa2, lambda: box3["o"][0])
except Exception as exc:
    rows.append({"impl": "flash_attn", "unavailable": str(exc)[:300]})

res = {"shape": {"n": args.n, "window": P, "heads": H, "kv_heads": G, "head_dim": D, "causal": True},
       "flops_causal_pairs": flops, "gpu": torch.cuda.get_device_name(), "rows": rows}
for r in rows:
    print(json.dumps(r))
if args.out:
    Path(args.out).write_text(json.dumps(res, indent=1))
