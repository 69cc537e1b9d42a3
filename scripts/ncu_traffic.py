"""DRAM traffic per launch of the evolve kernel from ncu --set full reports ->
profiles/traffic.json (read by bench.py for roofline.traffic).

    python scripts/ncu_traffic.py CONFIG REPORT.ncu-rep|RAW.csv [CONFIG REPORT ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_path = os.path.join(ROOT, "profiles", "traffic.json")
t = json.load(open(out_path)) if os.path.exists(out_path) else {}
args = sys.argv[1:]
for cfg, rep in zip(args[::2], args[1::2]):
    if rep.endswith(".csv"):   # an exported `--page raw --csv`
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "")
        if "evolve_brick_kernel" not in name:
            continue
        unit = dict(zip(h, u))

        def val(k):
            v = float(d[k].replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit[k]]
        b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        e = {"dram_bytes_per_launch": b, "dram_read": val("dram__bytes_read.sum"),
             "dram_write": val("dram__bytes_write.sum"), "kernel": name, "source": os.path.basename(rep)}
        # the binding units' speed-of-light percentages
        for key, metric in (("issue_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                            ("shared_wavefront_pct",
                             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                            ("l2_throughput_pct", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed"),
                            ("duration_ns", "gpu__time_duration.sum")):
            if metric in d and d[metric]:
                v = float(d[metric].replace(",", ""))
                if key == "duration_ns":
                    v *= {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}[unit[metric]]
                e[key] = v
        t.setdefault(cfg, {})["evolve_brick_kernel"] = e
        break
json.dump(t, open(out_path, "w"), indent=1)
print(json.dumps(t, indent=1))
