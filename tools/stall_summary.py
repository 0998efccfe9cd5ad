"""Warp-stall summary of one kernel from `ncu --page source --csv` output:
share of samples per stall reason and the instructions with the most samples.

    python tools/stall_summary.py gpurun_out/sweep_full_source.csv profiles/<name>.md
"""
import csv
import sys


def main(src, dst):
    rows = list(csv.reader(open(src)))
    name = rows[0][1] if len(rows[0]) > 1 else "?"
    h = rows[1]
    si, srci, ex = h.index("# Samples"), h.index("Source"), h.index("Instructions Executed")
    stall = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    data, agg, tot = [], {}, 0
    for r in rows[2:]:
        try:
            smp = int(r[si])
        except (ValueError, IndexError):
            continue
        tot += smp
        data.append((smp, r))
        for i in stall:
            agg[h[i]] = agg.get(h[i], 0) + int(r[i] or 0)
    out = [f"ncu --set full --import-source on, warp stall sampling of `{name}`", f"source: {src}", "",
           f"total samples: {tot}", "", "| stall reason | samples | share |", "|---|---|---|"]
    st = sum(agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
        out.append(f"| {k} | {v} | {100 * v / st:.1f}% |")
    out += ["", "| samples | share | executed | instruction | top stall |", "|---|---|---|---|---|"]
    for smp, r in sorted(data, key=lambda x: -x[0])[:25]:
        top = max(((int(r[i] or 0), h[i]) for i in stall), default=(0, ""))
        out.append(f"| {smp} | {100 * smp / max(tot, 1):.1f}% | {r[ex]} | `{r[srci].strip()[:70]}` | {top[1]} |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out[:20]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
