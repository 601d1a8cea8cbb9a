"""Per-barrier wait samples (SASS TRYWAIT lines + the spin branch after them) and the pipe summary of an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
hdr = rows[h]
si, src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
R = rows[h + 1:]
tot = 0.0
acc = {}
for k, r in enumerate(R):
    try:
        v = float(r[si])
    except (ValueError, IndexError):
        continue
    tot += v
    s = r[src]
    if "TRYWAIT" in s or "BAR.SYNC" in s or "BAR.RED" in s:
        key = s.split("[")[1].split("]")[0] if "[" in s else s.strip()[:30]
        w = v + (float(R[k + 1][si]) if k + 1 < len(R) else 0)
        acc[key] = acc.get(key, 0) + w
for k, v in sorted(acc.items(), key=lambda x: -x[1])[:16]:
    print(f"{v / tot:6.3f} {k}")
print("total samples", tot)
