"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel total
device time, launch count and share (cold-cache, serialised: compare shares only)."""
import collections
import csv
import sys


def main(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            agg[r[ki].split("(")[0][:70]].append(float(r[mi].replace(",", "")))
        except (ValueError, IndexError):
            pass
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':72s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:72s} {len(v):8d} {sum(v) / 1e6:10.3f} {sum(v) / len(v) / 1e3:10.2f} {100 * sum(v) / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
