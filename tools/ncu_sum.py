"""Summarise an ncu --csv metrics log per kernel: launches, total time, DRAM bytes.

    python tools/ncu_sum.py gpurun_out/launches.csv [--skip N]

--skip drops the first N launches (e.g. graph build / warm-up).
"""
import csv
import io
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = OrderedDict()
    ids = sorted({int(r["ID"]) for r in rows})
    keep = set(ids[skip:])
    for r in rows:
        if int(r["ID"]) not in keep:
            continue
        name = r["Kernel Name"].split("(")[0].replace("agpm_b200::<unnamed>::", "")
        d = per.setdefault(name, {"ids": set(), "ns": 0.0, "rd": 0.0, "wr": 0.0})
        d["ids"].add(r["ID"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        m = r["Metric Name"]
        if m == "gpu__time_duration.sum":
            d["ns"] += v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        elif m == "dram__bytes_read.sum":
            d["rd"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif m == "dram__bytes_write.sum":
            d["wr"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    total = sum(d["ns"] for d in per.values()) or 1.0
    print(f"{'kernel':60s} {'n':>5s} {'ms':>9s} {'share':>6s} {'rd GB':>8s} {'wr GB':>8s}")
    for name, d in sorted(per.items(), key=lambda kv: -kv[1]["ns"]):
        print(f"{name[:60]:60s} {len(d['ids']):5d} {d['ns'] / 1e6:9.3f} {d['ns'] / total:6.1%} "
              f"{d['rd'] / 1e9:8.3f} {d['wr'] / 1e9:8.3f}")
    print(f"{'total':60s} {'':5s} {total / 1e6:9.3f}")


if __name__ == "__main__":
    main()
