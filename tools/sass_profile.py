"""Summarise an ncu report's per-SASS-instruction counters (source page):
dynamic instruction mix per edge and stall reasons by opcode.

    python tools/sass_profile.py gpurun_out/prof_TAG.ncu-rep [edges_per_warp_iter_divisor]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 512 * 12 * 10 * 316
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r)
data = rows[rows.index(hdr) + 1:]
ie = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = {r: hdr.index(r) for r in reasons}
cnt = collections.Counter()
st = collections.Counter()
byop = collections.defaultdict(collections.Counter)
for r in data:
    if len(r) <= ie or not r[1].strip():
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).split()[0].split(".")[0]
    cnt[op] += int(r[ie] or 0)
    for k, i in ri.items():
        v = int(r[i] or 0)
        st[k] += v
        byop[op][k] += v
tot = sum(cnt.values())
print(f"instructions per edge-unit: {tot / div:.2f}")
for k, v in cnt.most_common(24):
    print(f"  {k:10s} {v / div:6.3f}")
T = sum(st.values())
print("stall reasons (share of samples):")
for k, v in st.most_common(12):
    top = sorted(((byop[o][k], o) for o in byop), reverse=True)[:4]
    print(f"  {k:24s} {100 * v / T:5.1f}%  top: " + ", ".join(f"{o} {100 * c / max(1, v):.0f}%" for c, o in top))
