"""Summarise an ncu launch list (CSV: gpu__time_duration.sum, optionally
dram__bytes_read.sum / dram__bytes_write.sum) per kernel: launches, total
time, share of the step, and DRAM GB/s where the byte counters are present."""
import collections
import csv
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, launches = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d.get("ID"), d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        launches.setdefault(key, {})[d["Metric Name"]] = v
    return launches


def main(path, skip_first=0):
    launches = list(load(path).items())[skip_first:]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in launches:
        k = name.split("(")[0].replace("void ", "").split("<")[0]
        agg[k][0] += 1
        agg[k][1] += m.get("gpu__time_duration.sum", 0.0)
        agg[k][2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':42s} {'launches':>8s} {'total us':>10s} {'share':>6s} {'us/launch':>10s} "
          f"{'DRAM MB/launch':>14s} {'DRAM GB/s':>10s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        per = v[1] / v[0]
        mb = v[2] / v[0] / 1e6
        gbs = v[2] / (v[1] * 1e-6) / 1e9 if v[1] > 0 else 0.0
        print(f"{k:42s} {v[0]:8d} {v[1]:10.1f} {100 * v[1] / tot:5.1f}% {per:10.1f} {mb:14.2f} "
              f"{gbs:10.1f}")
    print(f"{'TOTAL':42s} {len(launches):8d} {tot:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
