"""Aggregate executed warp-level instructions by CUDA source line from an ncu report (--page source)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ie = h.index("Instructions Executed")
cnt, src = defaultdict(float), {}
fname, cur = "", None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) <= ie or r[0] == "Line No":
        continue
    if r[0]:
        try:
            cur = (fname, int(r[0]))
            src[cur] = r[1].strip()[:80]
        except ValueError:
            pass
        continue
    try:
        cnt[cur] += float(r[ie] or 0)
    except ValueError:
        pass
T = sum(cnt.values())
print(f"total warp instructions {T:.4e}")
for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:top]:
    print(f"{k[0]}:{k[1]:<5d} {v:.3e} ({v / T:.1%}) | {src.get(k, '')}")
