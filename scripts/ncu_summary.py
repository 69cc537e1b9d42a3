"""Summarise ncu reports / launch lists into profiles/*.md (committed evidence).

    python scripts/ncu_summary.py REPORT.ncu-rep [...] --out profiles/x.md
    python scripts/ncu_summary.py --launches LAUNCHES.csv --out profiles/y.md
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Frequency", "Registers Per Thread",
        "Block Size", "Grid Size", "Dynamic Shared Memory Per Block", "Theoretical Occupancy",
        "Achieved Occupancy", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Issued Warp Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum",
       "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
       "smsp__thread_inst_executed_per_inst_executed.ratio"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    res = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0]
        res.setdefault(k, collections.OrderedDict())
        if r[mi] in KEYS and r[mi] not in res[k]:
            res[k][r[mi]] = f"{r[vi]} {r[ui]}".strip()
    return res


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in RAW:
            if m in hdr:
                d[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    tot, cnt = collections.OrderedDict(), collections.Counter()
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0, "s": 1e3}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
        tot[k] = tot.get(k, 0.0) + float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        cnt[k] += 1
    T = sum(tot.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / T:.2f}% |")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    md = [f"# {a.title}", ""]
    if a.launches:
        md += [f"## Launch list `{a.launches}` (cold-cache, serialised; compare shares)", "", launches(a.launches), ""]
    for rep in a.reports:
        md += [f"## `{rep}`", ""]
        for k, m in details(rep).items():
            md += [f"### {k}", "", "| metric | value |", "|---|---|"] + [f"| {x} | {v} |" for x, v in m.items()] + [""]
        rr = raw(rep)
        if rr:
            md += ["raw counters:", "", "| kernel | " + " | ".join(RAW) + " |",
                   "|---|" + "---|" * len(RAW)]
            for d in rr:
                md.append(f"| {d['kernel']} | " + " | ".join(d.get(m, "") for m in RAW) + " |")
            md.append("")
    open(a.out, "w").write("\n".join(md) + "\n")
    print(a.out)


if __name__ == "__main__":
    main()
