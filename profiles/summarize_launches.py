"""Summarise an ncu --metrics launch list (CSV) per kernel: count, mean time,
DRAM bytes, share of the step.  Usage: python summarize_launches.py file.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0]
        try:
            v = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = d["Metric Unit"]
        if unit == "ns":
            v /= 1e3
        elif unit == "us":
            pass
        elif unit == "ms":
            v *= 1e3
        elif unit in ("byte", "Kbyte", "Mbyte", "Gbyte"):
            v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}[unit]
        per[name][d["Metric Name"]].append(v)
    total = sum(sum(m.get("gpu__time_duration.sum", [])) for m in per.values())
    print(f"{'kernel':32s} {'n':>5s} {'mean_us':>9s} {'share':>6s} {'MB_read':>9s} {'GB/s':>8s}")
    for k, m in sorted(per.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", []))):
        t = m.get("gpu__time_duration.sum", [])
        b = m.get("dram__bytes_read.sum", [])
        mt = sum(t) / len(t) if t else 0
        mb = sum(b) / len(b) if b else 0
        print(f"{k:32s} {len(t):5d} {mt:9.2f} {sum(t)/total:6.1%} {mb:9.1f} {mb/mt*1e3 if mt else 0:8.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
