"""Top source lines by executed instructions / stall samples from an ncu
report (cuda view). Usage: python tools/src_lines.py REP [file-substring] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, i_s, i_i, i_src = None, None, None, None
res = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1]
        continue
    if r[0] == "Line No":
        i_s = r.index("Warp Stall Sampling (All Samples)")
        i_i = r.index("Instructions Executed")
        i_src = 1
        continue
    if i_s is None or not r[0].strip().isdigit() or sub not in (cur or ""):
        continue
    try:
        res.append((float(r[i_i] or 0), float(r[i_s] or 0), cur.rsplit("/", 1)[-1], int(r[0]), r[i_src].strip()[:90]))
    except ValueError:
        pass
ti = sum(x[0] for x in res) or 1
ts = sum(x[1] for x in res) or 1
for x in sorted(res, reverse=True)[:top]:
    print(f"{100 * x[0] / ti:5.1f}% inst {100 * x[1] / ts:5.1f}% samp  {x[2]}:{x[3]}  {x[4]}")
