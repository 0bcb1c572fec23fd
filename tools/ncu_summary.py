"""Summarise ncu reports (raw page) into profiles/: a markdown table per kernel and the
residue-GEMM DRAM traffic JSON that bench.py reports as roofline.traffic.

    python tools/ncu_summary.py gpurun_out/prof16k.ncu-rep profiles/round1_ncu_16k.md \
        [--traffic-json profiles/ncu_residue_gemm.json --m 16384 --N 13]
"""
import argparse
import csv
import io
import json
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long-sb"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math-throttle"),
]


def load(rep):
    if rep.endswith(".csv"):          # `ncu -i rep --page raw --csv` output saved on the box
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(io.StringIO(out)) if r]
    while rows and rows[0][0] != "ID":
        rows = rows[1:]
    h, units = rows[0], rows[1]
    return h, units, rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out_md")
    ap.add_argument("--traffic-json")
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--N", type=int, default=13)
    ap.add_argument("--title", default="")
    ap.add_argument("--scheme", default="fp8")
    a = ap.parse_args()
    h, units, rows = load(a.rep)
    lines = [f"# ncu summary {a.title}", "", f"source: `{a.rep}` (ncu --set full --clock-control none)", ""]
    cols = [(h.index(k), lbl, units[h.index(k)]) for k, lbl in METRICS if k in h]
    lines.append("| kernel | " + " | ".join(f"{lbl} [{u}]" if u else lbl for _, lbl, u in cols) + " |")
    lines.append("|---" * (len(cols) + 1) + "|")
    res = None
    for r in rows:
        name = r[h.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "")
        lines.append(f"| `{short}` | " + " | ".join(r[i] for i, _, _ in cols) + " |")
        if ("gemm_kernel<0" in name or "gemm_kernel<3" in name) and res is None:
            res = r
    with open(a.out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic_json and res is not None:
        def val(k):
            i = h.index(k)
            v = float(res[i].replace(",", ""))
            u = units[i]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
            return v * scale
        tr = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        with open(a.traffic_json, "w") as f:
            json.dump({"kernel": res[h.index("Kernel Name")].split("(")[0], "m": a.m, "num_moduli": a.N,
                       "scheme": a.scheme,
                       "dram_bytes_per_launch": tr, "source": a.rep}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
