"""Per-kernel launch count, time and share of an ncu launch list
(ncu --metrics gpu__time_duration.sum --csv --log-file LIST.csv CMD).

    python tools/launch_summary.py LIST.csv "header note" > summary.txt
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def main(path, note=""):
    lines = open(path).read().splitlines()
    start = next(k for k, line in enumerate(lines) if line.startswith('"ID"'))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for x in csv.DictReader(lines[start:]):
        if x.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ms = float(x["Metric Value"].replace(",", "")) * SCALE[x["Metric Unit"]]
        name = x["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(a[1] for a in agg.values()) or 1.0
    print(f"# ncu launch list {path}: serialised, cold-cache launches (compare shares, not absolutes) {note}".rstrip())
    print(f"{'kernel':60s} {'launches':>8s} {'ms':>11s} {'share':>7s}")
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {n:8d} {ms:11.3f} {100 * ms / tot:6.2f}%")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
