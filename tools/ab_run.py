"""Same-box A/B of library builds: runs `cmd` with DS_LIB=<each .so>, interleaved
for --rounds rounds, and prints the last line of each run.

    python tools/ab_run.py --rounds 3 --cmd "python tools/attn_bench.py" ab/a.so ab/b.so
"""
import argparse
import os
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--cmd", required=True)
ap.add_argument("libs", nargs="+")
args = ap.parse_args()
for r in range(args.rounds):
    for lib in args.libs:
        env = dict(os.environ, DS_LIB=os.path.abspath(lib))
        out = subprocess.run(args.cmd, shell=True, env=env, capture_output=True, text=True)
        lines = [l for l in (out.stdout + out.stderr).splitlines() if l.strip()]
        print(f"round {r} {os.path.basename(lib)}: {lines[-1] if lines else '(no output)'}", flush=True)
