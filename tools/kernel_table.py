"""Per-kernel table (duration, DRAM bytes, achieved GB/s vs the measured copy
peak) from an ncu report: python tools/kernel_table.py REP OUT.md"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, dst):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, rows = r[0], r[1], r[2:]
    bs = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    ts = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}

    def val(v, n, sc):
        return float(v[h.index(n)].replace(",", "")) * sc.get(u[h.index(n)], 1)

    peak = 6443.8
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
                     .get("hbm_gbs", peak))
    except Exception:
        pass
    agg = {}
    for v in rows:
        name = v[h.index("Kernel Name")].split("(")[0].replace("eqb::<unnamed>::", "")
        name = name.replace("void ", "")[:60]
        t = val(v, "gpu__time_duration.sum", ts)
        by = val(v, "dram__bytes_read.sum", bs) + val(v, "dram__bytes_write.sum", bs)
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += t
        a[2] += by
    out = ["| kernel | launches | avg time | avg DRAM bytes | DRAM GB/s | frac of peak |",
           "|---|---|---|---|---|---|"]
    for name, (c, t, by) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = by / t / 1e9 if t > 0 else 0.0
        out.append(f"| {name} | {c} | {t / c * 1e6:.1f} us | {by / c / 1e6:.1f} MB | "
                   f"{gbs:.0f} | {gbs / peak:.2f} |")
    with open(dst, "w") as f:
        f.write(f"ncu (cold-cache, serialised, --clock-control none) over tools/kernels_prof.py: "
                f"dense c2 SGD, c4 LSQR and c3 setup + SGD kernels; DRAM GB/s is measured "
                f"traffic / duration, peak {peak} GB/s (MEASURED_PEAKS.json copy bandwidth)\n"
                f"source: {rep}\n\n" + "\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
