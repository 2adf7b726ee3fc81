"""Summarise tools/raster_sweep.sh output: median DRAM read/write MB, L2 GB and
ncu time per recompute GEMM shape for each setting."""
import collections
import csv
import glob
import sys

for path in sorted(glob.glob("gpurun_out/raster_time_*.txt"), key=lambda p: int(p.split("_")[-1][:-4])):
    i = path.split("_")[-1][:-4]
    label = open(path).readline().strip()
    try:
        rows = list(csv.DictReader(l for l in open(f"gpurun_out/raster_{i}.csv") if not l.startswith("==")))
    except OSError:
        continue
    by = collections.defaultdict(dict)
    for r in rows:
        by[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ids = sorted(by, key=int)
    per = len(ids) // 4
    out = []
    for s in range(4):
        sel = [by[j] for j in ids[s * per:(s + 1) * per]]
        med = lambda k: sorted(x[k] for x in sel)[len(sel) // 2]  # noqa: E731
        out.append(f"{['qkv', 'o', 'w1', 'w2'][s]} rd {med('dram__bytes_read.sum') / 1e6:.0f} "
                   f"wr {med('dram__bytes_write.sum') / 1e6:.0f} MB {med('gpu__time_duration.sum') / 1e3:.1f}us")
    times = [l.split(":")[-1].strip() for l in open(path).read().splitlines()[1:] if "TFLOP" in l]
    print(f"{label:45s} | " + " | ".join(out))
    print(f"{'':45s} | events: " + " | ".join(times))
