"""Summarise ncu output into profiles/ (committed evidence).

    python tools/summarize_ncu.py launches  gpurun_out/launches.csv  profiles/<round>_launches.md
    python tools/summarize_ncu.py full      gpurun_out/prof.ncu-rep  profiles/<round>_sgd_iter_full.md

'full' also writes profiles/ncu_summary.json, which bench.py reads for the
roofline "traffic" field (dram read+write bytes per sgd_iter_kernel launch).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(src, dst):
    rows = [r for r in csv.reader(open(src)) if len(r) > 5]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    total = 0.0
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("eqb::<unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
        total += ns
    out = ["| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {name[:70]} | {c} | {t / 1e6:.3f} | {t / c / 1e3:.2f} | {100 * t / total:.1f}% |")
    with open(dst, "w") as f:
        f.write(f"ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, "
                f"serialised; compare shares)\nsource: {src}\n\n" + "\n".join(out) + "\n")
    print("\n".join(out))


def full(rep, dst):
    """One ncu --set full capture of the launches of ONE SGD iteration (the
    long-row and slice parts of sgd_iter_kernel); per-launch metrics and the
    per-iteration DRAM traffic (sum over the parts)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, rows = r[0], r[1], r[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tscale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1, "ms": 1}

    def get(v, n, sc):
        if n not in h:
            return 0.0
        return float(v[h.index(n)].replace(",", "")) * sc.get(u[h.index(n)], 1)

    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
            "lts__t_sectors_srcunit_tex_op_read.sum"]
    names = [v[h.index("Kernel Name")][:40] if "Kernel Name" in h else f"launch {k}"
             for k, v in enumerate(rows)]
    lines = ["| metric | " + " | ".join(names) + " |", "|---|" + "---|" * len(rows)]
    for k in keys:
        if k in h:
            lines.append(f"| {k} ({u[h.index(k)]}) | " +
                         " | ".join(v[h.index(k)] for v in rows) + " |")
    rd = sum(get(v, "dram__bytes_read.sum", scale) for v in rows)
    wr = sum(get(v, "dram__bytes_write.sum", scale) for v in rows)
    dur = sum(get(v, "gpu__time_duration.sum", tscale) for v in rows)
    with open(dst, "w") as f:
        f.write(f"ncu --set full --clock-control none: the {len(rows)} launches of one SGD "
                f"iteration on c3 (serialised by ncu)\nsource: {rep}\n\n" +
                "\n".join(lines) + f"\n\nper iteration: DRAM {rd / 1e9:.3f} GB read + "
                f"{wr / 1e9:.3f} GB written, {dur:.3f} ms summed\n")
    summ = os.path.join(ROOT, "profiles", "ncu_summary.json")
    d = {}
    if os.path.exists(summ):
        d = json.load(open(summ))
    d["sgd_iter_kernel"] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd,
                            "dram_write": wr, "duration_ms": dur, "launches": len(rows),
                            "source": dst}
    json.dump(d, open(summ, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
