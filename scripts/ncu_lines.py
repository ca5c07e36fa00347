"""Per-source-line instruction and stall totals of one ncu report
(ncu -i REP --page source --csv --print-source cuda,sass).

    python scripts/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
fname = "?"
h = None
cur = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = {k: i for i, k in enumerate(r)}
        continue
    if h is None or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1][:90])
        continue
    if cur is None:
        continue
    num = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
    a = agg.setdefault(cur, [0.0, 0.0])
    a[0] += num(r[7])          # Instructions Executed (warp level)
    a[1] += num(r[4])          # stall samples
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]/tot_i*100:5.1f}% inst {v[1]/tot_s*100:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
