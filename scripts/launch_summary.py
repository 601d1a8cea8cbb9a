"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel: count, total us, share."""
import collections
import csv
import sys


def main(path, top=20):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[r[ki][:70]][0] += 1
        agg[r[ki][:70]][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total_us':>10} {'avg_us':>9} {'share':>6}  kernel   ({path})")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v[0]:8d} {v[1] / 1e3:10.1f} {v[1] / 1e3 / v[0]:9.2f} {v[1] / tot:6.3f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
