"""Calibrate the reference planner's cost model (sched.py:86-104) on measured
B200 times and check its TTFT predictions (estimate_ttft, sched.py:279-281)
against measured consumer TTFTs; then let adapt_config (sim.py:171-202) pick a
recompute set per SLO with the calibrated model.

Calibration (one run at k = 6): per-layer recompute time = recompute group
alone / 6; the anchor's cost = what the fused step adds over the recompute
(the anchor runs beside it; only its tail is exposed); link = HBM (the
producer export is on this GPU; the ingest is fused into the anchor).

    python tools/costmodel_check.py [--n 8192] > profiles/r01_costmodel.json
"""
import argparse
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2411_02820_b200 as P  # noqa: E402
from paper_2411_02820_b200 import _lib as L, planner as S, selection as SEL  # noqa: E402
from paper_2411_02820_b200.engine import _workspace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--ks", default="3,6,10,13,16")
args = ap.parse_args()
ks = [int(x) for x in args.ks.split(",")]
cfg = P.ModelConfig(32, 4096, 32, 8, 128, 14336, 128256, args.n + 64, 0)
Ln, n = cfg.n_layers, args.n
A = P.random_model(cfg, seed=1000)
B = P.random_model(cfg, seed=2000, base=A, perturb_layers=range(Ln - max(ks), Ln))
ids = np.random.default_rng(7).integers(0, cfg.vocab_size, size=n, dtype=np.int64)
tok = torch.from_numpy(ids).cuda()
prod = P.full_prefill(A, ids, e_layers=[Ln - k for k in ks], tokens_dev=tok)
cache = P.PagedKV.allocate(cfg, n)
s, side = torch.cuda.Stream(), torch.cuda.Stream()
lib = L.lib()


def graph_ms(fn, reps=15):
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    ts = []
    for _ in range(3 + reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        with torch.cuda.stream(s):
            g.replay()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[3:])


measured = {}
for k in ks:
    rc = P.RecomputeConfig([(Ln - k, Ln - 1)])
    measured[k] = graph_ms(lambda: P.partial_prefill(B, ids, rc, prod.kv, prod.e_map(), out=cache, stream=s,
                                                     copy_stream=side, tokens_dev=tok))
ws = _workspace(B, n, s)
e6 = prod.e_map()[Ln - 6].hidden
d = cache.desc()
rec6 = graph_ms(lambda: L.check(lib.ds_recompute_group(C.byref(B.desc()), tok.data_ptr(), n, Ln - 6, Ln - 1,
                                                       e6.data_ptr(), e6.shape[0], C.byref(d), ws.data_ptr(),
                                                       ws.numel(), s.cuda_stream)))
layer_ms = rec6 / 6
anchor_ms = measured[6] - rec6
hbm = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6500.0) \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6500.0
cost = S.CostModel.from_measured(cfg, n - 1, hbm, layer_ms, anchor_ms)
rows = []
for k in ks:
    req = S.ScheduledRequest("r", 0.0, "B", P.RecomputeConfig([(Ln - k, Ln - 1)]), Ln)
    pred = S.estimate_ttft(req, cost)
    rows.append({"k": k, "measured_ms": round(measured[k], 3), "predicted_ms": round(pred, 3),
                 "error": round((pred - measured[k]) / measured[k], 4)})
# adapt_config with the calibrated model over a frontier whose quality grows with k
pts = [SEL.ProfilePoint(P.RecomputeConfig([(Ln - k, Ln - 1)]), k, min(1.0, 0.5 + k / 32)) for k in range(1, Ln)]
pts.append(SEL.ProfilePoint(P.RecomputeConfig.full(Ln), Ln, 1.0))
fr = SEL.build_frontier(pts)
req = S.ScheduledRequest("r", 0.0, "B", P.RecomputeConfig.full(Ln), Ln)
choices = []
for slo in (12.0, 16.0, 20.0, 30.0, 60.0):
    for qd in (0, 2):
        dec = S.adapt_config(qd, req, fr, S.SloPolicy(slo, 0.6), cost)
        choices.append({"slo_ms": slo, "queue_depth": qd, "k": dec.k, "quality": dec.quality,
                        "slo_feasible": dec.slo_feasible})
print(json.dumps({"n": n, "calibration": {"recompute_k6_ms": round(rec6, 3), "layer_ms": round(layer_ms, 4),
                                          "anchor_exposed_ms": round(anchor_ms, 3), "link_gbs": hbm},
                  "ttft": rows, "adapt_config": choices}, indent=1))
