"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per kernel
name, launches, mean and total us, in first-seen order (optionally only the
launches with ID in [lo, hi))."""
import csv
import sys
from collections import OrderedDict


def main(path, lo=0, hi=1 << 60):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum" or not (lo <= int(d["ID"]) < hi):
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("hetm_b200::", "")
        ns = float(d["Metric Value"]) * (1e3 if d.get("Metric Unit") == "usecond" else 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    print(f"{'kernel':60s} {'n':>4s} {'mean us':>9s} {'total us':>10s}")
    for k, (n, t) in agg.items():
        print(f"{k[:60]:60s} {n:4d} {t / n / 1e3:9.2f} {t / 1e3:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(x) for x in sys.argv[2:4]))
