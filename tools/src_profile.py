#!/usr/bin/env python
"""Share of warp-stall samples and executed instructions per source function,
from an ncu report's cuda,sass source view (compile with -lineinfo,
capture with --import-source on).

    python tools/src_profile.py REP [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


samp, inst = collections.Counter(), collections.Counter()
cur_file, i_s, i_i = None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] == "Line No":
        i_s = r.index("Warp Stall Sampling (All Samples)")
        i_i = r.index("Instructions Executed")
        continue
    if i_s is None or len(r) <= i_s or not r[0].strip().isdigit():
        continue
    key = (cur_file, int(r[0]))
    samp[key] += num(r[i_s])
    inst[key] += num(r[i_i])

funcs = collections.defaultdict(list)
for path in {k[0] for k in samp}:
    try:
        lines = open(path).read().split("\n")
    except OSError:
        continue
    for i, line in enumerate(lines, 1):
        if ("__device__" in line or "__global__" in line) and "(" in line:
            names = [n for n in re.findall(r"(\w+)\s*\(", line) if n not in ("__launch_bounds__", "constexpr")]
            if names:
                funcs[path].append((i, names[0]))


def func_of(path, line):
    if "/paper_2009_05534_b200/" not in path:
        return "[" + path.rsplit("/", 1)[-1] + "]"  # CUDA header intrinsics (half2 arithmetic etc.)
    best = "?"
    for s, n in funcs.get(path, []):
        if s <= line:
            best = n
    return best


agg_s, agg_i = collections.Counter(), collections.Counter()
for (path, line), v in samp.items():
    agg_s[func_of(path, line)] += v
for (path, line), v in inst.items():
    agg_i[func_of(path, line)] += v
ts, ti = sum(agg_s.values()) or 1, sum(agg_i.values()) or 1
print(f"{'function':28s} {'samples':>8s} {'instr':>8s}")
for n, v in agg_s.most_common(top):
    print(f"{n:28s} {100 * v / ts:7.1f}% {100 * agg_i[n] / ti:7.1f}%")
