"""Summarise ncu outputs into profiles/ (run in the build container).

    python tools/ncu_summary.py launches <launches.csv>      per-kernel share of a step
    python tools/ncu_summary.py full <report.ncu-rep>        per-launch time / DRAM bytes / SM+tensor %
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1, "second": 1}


def launches(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows:
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        tot[k] += float(r["Metric Value"]) * UNIT.get(r["Metric Unit"], 1e-9) * 1e3
        cnt[k] += 1
    T = sum(tot.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total_ms':>9s} {'share':>6s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:44s} {cnt[k]:8d} {v:9.3f} {v / T:6.3f}")
    print(f"{'TOTAL (serialised, cold-cache)':44s} {sum(cnt.values()):8d} {T:9.3f}")


FULL = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path):
    """A .ncu-rep (read with ncu -i) or its --page raw --csv export."""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units = r[0], r[1]
    have = [m for m in FULL if m in head]
    extra = [h for h in head if "tensor" in h and "pct" in h and h not in have][:4]
    cols = have + extra
    print("kernel | " + " | ".join(cols))
    for row in r[2:]:
        vals = []
        for m in cols:
            i = head.index(m)
            u = units[i]
            v = row[i]
            if m.startswith("dram__bytes"):
                v = f"{float(v.replace(',', '')) * UNIT.get(u, 1) / 1e6:.1f} MB"
            elif m == "gpu__time_duration.sum":
                v = f"{float(v.replace(',', '')) * UNIT.get(u, 1) * 1e3:.4f} ms"
            vals.append(v)
        print(row[head.index("Kernel Name")].split("(")[0].replace("void ", "") + " | " + " | ".join(vals))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
