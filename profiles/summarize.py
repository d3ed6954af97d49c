"""Summarise ncu reports into profiles/<round>_ncu_summary.md (run here, no GPU).

usage: python profiles/summarize.py <round> <launches.csv> <report.ncu-rep> [<report.ncu-rep> ...]
"""
import collections
import csv
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instr"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui] if ui is not None else ""
        v = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
        name = r[ki].split("(")[0].replace("void ", "")[:48]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    return agg


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m, label in METRICS:
            if m in h:
                d[label] = (r[h.index(m)], units[h.index(m)])
        res.append(d)
    return res


def main():
    rnd, lpath, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    here = os.path.dirname(os.path.abspath(__file__))
    lines = [f"# ncu summary ({rnd})", "", f"Launch list: `{os.path.basename(lpath)}` "
             "(`ncu --metrics gpu__time_duration.sum --clock-control none`, cold-cache and serialised: "
             "compare shares, not absolutes). Dataset-generation kernels (k_rmat, k_features, CUB sort/select, "
             "k_indptr_from_sorted) are setup, outside the timed step.", "",
             "| kernel | launches | total µs | avg µs |", "|---|---:|---:|---:|"]
    for k, (n, t) in sorted(launches(lpath).items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {n} | {t:.1f} | {t / n:.1f} |")
    traffic = {}
    for rp in reps:
        lines += ["", f"## `{os.path.basename(rp)}` (`ncu --set full`)", ""]
        rs = report(rp)
        labels = [l for _, l in METRICS]
        lines.append("| kernel | " + " | ".join(labels) + " |")
        lines.append("|---|" + "---|" * len(labels))
        for d in rs:
            lines.append(f"| {d['kernel'][:40]} | " + " | ".join(
                f"{d[l][0]} {d[l][1]}".strip() if l in d else "" for l in labels) + " |")
            if ("gather" in d["kernel"] or "fan_rows" in d["kernel"]) and "DRAM read" in d:
                def mb(x):
                    v, u = float(x[0]), x[1]
                    return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1)
                traffic.setdefault(d["kernel"], []).append(mb(d["DRAM read"]) + mb(d["DRAM write"]))
    with open(os.path.join(here, f"{rnd}_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    for k, v in traffic.items():
        print(k, sum(v) / len(v))
    if traffic:
        out = {"source": [os.path.basename(r) for r in reps]}
        for key, pre in (("k_gather", "k_gather_tma2"), ("k_fan", "k_fan_rows")):
            k = next((x for x in traffic if x.startswith(pre)), None)
            if k:
                out[key + "_kernel"] = k
                out[key + "_dram_bytes_per_launch"] = sum(traffic[k]) / len(traffic[k])
                out[key + "_launches_captured"] = len(traffic[k])
        json.dump(out, open(os.path.join(here, "traffic_papers.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
