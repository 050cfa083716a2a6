"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys


def main(path, header=""):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = row["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(row["Metric Value"].replace(",", ""))
        unit = row["Metric Unit"]
        ms = v / 1e6 if unit in ("ns", "nsecond") else v / 1e3 if unit in ("us", "usecond") else v
        tot[name] += ms
        cnt[name] += 1
    T = sum(tot.values()) or 1.0
    if header:
        print(header)
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:60s} n={cnt[k]:5d} total={tot[k]:9.3f} ms share={100 * tot[k] / T:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
