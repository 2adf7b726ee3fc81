"""Per-kernel SASS instruction counts proving the sm_100a features (run in the build container):
UTCHMMA / UTCQMMA (tcgen05.mma), UTCBAR (tcgen05.commit), LDTM / STTM (tcgen05.ld / st), UTMALDG (TMA tensor
load), UBLKCP (cp.async.bulk), SYNCS (mbarrier), FFMA2 / FADD2 (packed fp32), MUFU.EX2.

    python tools/sass_evidence.py > profiles/r02_sass_evidence.txt
"""
import collections
import re
import subprocess
from pathlib import Path

BUILD = Path(__file__).resolve().parents[1] / "paper_2411_02820_b200" / "build"
OPS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UBLKCP", "SYNCS", "FFMA2", "FADD2", "MUFU.EX2", "HMMA"]
print("# cuobjdump -sass of the in-tree build (sm_100a); instruction counts per kernel")
print("kernel | " + " | ".join(OPS))
for obj in sorted(BUILD.glob("*.o")):
    sass = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True).stdout
    cur, counts = None, collections.OrderedDict()
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        for op in OPS:
            if re.search(r"\b" + re.escape(op) + r"\b", line):
                counts[cur][op] += 1
    for fn, c in counts.items():
        if not any(c[o] for o in ("UTCHMMA", "LDTM", "UTMALDG", "UBLKCP", "FFMA2", "MUFU.EX2")):
            continue
        name = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(.*", "", name).replace("void ", "")
        print(f"{obj.stem}:{name} | " + " | ".join(str(c[o]) for o in OPS))
