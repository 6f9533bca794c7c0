"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list into per-kernel shares."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
            name = d["Kernel Name"].split("(")[0][:60]
            tot[name] += v
            cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:60s} {cnt[k]:8d} {v:10.1f} {100 * v / s:6.1f}%")
    print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {s:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
