"""Aggregate ncu --page source (cuda,sass) CSV by CUDA source line: warp-stall samples and top stall reasons."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr_i]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = defaultdict(float)
reasons = defaultdict(lambda: defaultdict(float))
src = {}
cur = None
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) <= si or r[0] == "Line No":
        continue
    if r[0]:
        try:
            cur = (fname, int(r[0]))
        except ValueError:
            continue
        src[cur] = r[1]
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    if cur is None:
        continue
    tot[cur] += v
    for c in stall_cols:
        try:
            reasons[cur][h[c]] += float(r[c] or 0)
        except ValueError:
            pass
S = sum(tot.values())
print(f"total samples {S:.0f}")
for ln in sorted(tot, key=lambda k: -tot[k])[:top]:
    rs = sorted(reasons[ln].items(), key=lambda kv: -kv[1])[:3]
    print(f"{ln[0][:12]}:{ln[1]:<4d} {tot[ln] / S * 100:5.1f}%  {', '.join(f'{k[6:]}={v / max(tot[ln], 1) * 100:.0f}%' for k, v in rs):55s} | {src.get(ln, '').strip()[:70]}")
