"""Per-kernel device time from an ncu launch list (gpu__time_duration.sum CSV)."""
import csv
import collections
import sys


def main(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        tot[name] += v
        cnt[name] += 1
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:40s} n={cnt[k]:5d} total={tot[k]:9.3f} ms  mean={tot[k]/cnt[k]:8.4f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
