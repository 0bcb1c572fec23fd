"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into markdown."""
import csv
import sys


def main(src, dst, title):
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
    tot, order = {}, []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        if name not in tot:
            order.append(name)
        tot.setdefault(name, []).append(v)
    ours = [n for n in order if n.startswith("oz2::")]
    total = sum(sum(tot[n]) for n in ours)
    lines = [f"# {title}", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: "
             "compare shares, not absolutes).", "",
             "| kernel | launches | mean ms | total ms | share of our kernels |", "|---|---|---|---|---|"]
    for n in sorted(ours, key=lambda n: -sum(tot[n])):
        v = tot[n]
        lines.append(f"| `{n}` | {len(v)} | {sum(v) / len(v):.3f} | {sum(v):.2f} | {sum(v) / total:.1%} |")
    others = [n for n in order if n not in ours]
    lines += ["", f"{len(others)} other (torch input generation) kernels, outside the timed steps."]
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
