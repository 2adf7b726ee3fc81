"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys

UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
for f in sys.argv[1:]:
    lines = [l for l in open(f) if not l.startswith("==")]
    t, c = collections.defaultdict(float), collections.Counter()
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("void ", "")[:50]
        t[k] += float(r["Metric Value"]) * UNIT.get(r["Metric Unit"], 1e-9) * 1e6
        c[k] += 1
    print(f"{f}: total {sum(t.values()):.0f} us")
    for k in sorted(t, key=lambda x: -t[x]):
        print(f"  {k:50s} n={c[k]:4d} {t[k]:9.1f} us  per-launch {t[k] / c[k]:.2f} us")
