"""Summarise ncu captures into the committed profiles/ evidence.

    python profiles/summarize.py full <report.ncu-rep> <out.md> [pairs_per_launch]
    python profiles/summarize.py launches <launches.csv> <out.md>
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 wavefronts %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def full(rep, out, pairs=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, units = r[0], r[1]
    stall = [(i, n) for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
    lines = [f"# ncu --set full summary: `{rep}`", ""]
    js = []
    for row in r[2:]:
        name = row[h.index("Kernel Name")].split("(")[0]
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        d = {"kernel": name}
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"| {label} (`{k}`) | {row[i]} | {units[i]} |")
                d[k] = row[i]
        top = sorted(((float(row[i] or 0), n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")) for i, n in stall), reverse=True)[:6]
        lines.append("")
        lines.append("Top stall reasons (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in top))
        lines.append("")
        js.append(d)
    open(out, "w").write("\n".join(lines) + "\n")
    ks = [d for d in js if "keyswitch" in d["kernel"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    unit = units[h.index("dram__bytes_read.sum")]
    if ks and pairs:
        rd = float(ks[0]["dram__bytes_read.sum"]) * scale[unit]
        wr = float(ks[0]["dram__bytes_write.sum"]) * scale[units[h.index("dram__bytes_write.sum")]]
        json.dump({"source": rep, "kernel": ks[0]["kernel"], "pairs_per_launch": pairs,
                   "dram_bytes_per_launch": rd + wr, "dram_bytes_per_pair": (rd + wr) / pairs},
                  open(out.rsplit("/", 1)[0] + "/keyswitch_traffic.json", "w"), indent=1)


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            v = v / 1000 if r[ui] == "ns" else (v * 1000 if r[ui] == "ms" else v)
            agg[r[ki].split("(")[0].split("::")[-1]].append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none): `{path}`", "",
             "Cold-cache, serialised launches: compare shares, not absolute times.", "",
             "| kernel | launches | avg us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {sum(v)/tot:.3f} |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
