"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]):
per kernel (template args kept short) launches, total / avg time, DRAM bytes.
python tools/launch_summary.py LAUNCHES.csv [skip_first_n]"""
import csv
import re
import sys
from collections import OrderedDict


def short(name):
    name = name.replace("eqb::<unnamed>::", "").replace("void ", "")
    m = re.match(r"([\w:]+)(<[^()]*>)?", name)
    base = m.group(1) if m else name
    tmpl = m.group(2) or "" if m else ""
    tmpl = re.sub(r"eqb::<unnamed>::", "", tmpl)
    tmpl = re.sub(r"\(\w+\)", "", tmpl)
    return (base + tmpl)[:90]


def main(path, skip=0):
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    per = OrderedDict()
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        d = per.setdefault(key, {})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            v *= {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6,
                  "ms": 1e-3, "msecond": 1e-3}.get(unit, 1)
        else:
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        d[r["Metric Name"]] = v
    items = list(per.items())[skip:]
    agg = OrderedDict()
    tot = 0.0
    for (i, name), d in items:
        a = agg.setdefault(short(name), [0, 0.0, 0.0])
        t = d.get("gpu__time_duration.sum", 0.0)
        a[0] += 1
        a[1] += t
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        tot += t
    print(f"{len(items)} launches, {tot * 1e3:.3f} ms total")
    print("| kernel | launches | total ms | avg us | share | avg DRAM MB |")
    print("|---|---|---|---|---|---|")
    for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {c} | {t * 1e3:.3f} | {t / c * 1e6:.1f} | {t / tot:.3f} | {b / c / 1e6:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
