"""Aggregate excessive shared-memory wavefronts (bank conflicts) by CUDA source line from an ncu report."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ex, wf = h.index("L1 Wavefronts Shared Excessive"), h.index("L1 Wavefronts Shared")
exc, tot, src = defaultdict(float), defaultdict(float), {}
fname, cur = "", None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) <= wf or r[0] == "Line No":
        continue
    if r[0]:
        try:
            cur = (fname, int(r[0]))
            src[cur] = r[1].strip()[:70]
        except ValueError:
            pass
        continue
    try:
        exc[cur] += float(r[ex] or 0)
        tot[cur] += float(r[wf] or 0)
    except ValueError:
        pass
T = sum(exc.values())
print(f"total excessive wavefronts {T:.3e}, total shared wavefronts {sum(tot.values()):.3e}")
for k, v in sorted(exc.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{k[0]}:{k[1]:<5d} excess {v:.3e} ({v / max(T, 1):.1%}) of {tot[k]:.3e} | {src.get(k, '')}")
