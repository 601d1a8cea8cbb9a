"""Top SASS instructions by warp-stall samples from an ncu report (--page source, SASS view)."""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
    hdr = rows[hdr_i]
    si, src, ai = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Address")
    data = []
    for k, r in enumerate(rows[hdr_i + 1:]):
        try:
            data.append((float(r[si]), k, r[ai][-5:], r[src].strip()[:90]))
        except (ValueError, IndexError):
            continue
    tot = sum(d[0] for d in data) or 1
    for v, k, a, s in sorted(data, reverse=True)[:top]:
        print(f"{v / tot:6.3f} #{k:5d} {a} {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
