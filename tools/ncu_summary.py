#!/usr/bin/env python3
"""Summarise ncu captures brought back in gpurun_out/ into profiles/.

    python tools/ncu_summary.py ROUND CONFIG PREC POINTS [CONFIG PREC POINTS ...]

For each (config, prec) it reads
  gpurun_out/prof_<config>_<prec>.ncu-rep   (`ncu --set full`, 1 launch)
  gpurun_out/launches_<config>_<prec>.csv   (launch list: duration + DRAM bytes)
and writes profiles/<round>_<config>_<prec>.json (key metrics, stall
reasons, launch list) and updates profiles/traffic.json, which bench.py
reads for the roofline `traffic` field.  POINTS is the --n the capture ran.
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__maximum_warps_per_active_cycle_pct",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_bytes_pipe_lsu_mem_global_op_st.sum",
]


def raw(rep):
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    stalls = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            out[h] = {"value": v, "unit": u}
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                n = float(v.replace(",", ""))
            except ValueError:
                continue
            if n > 0:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = n
    out["kernel"] = dict(zip(hdr, vals)).get("Kernel Name", "")
    return out, dict(sorted(stalls.items(), key=lambda kv: -kv[1]))


def launches(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    per = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"][:90])
        per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [{"id": int(k[0]), "kernel": k[1], **v} for k, v in sorted(per.items(),
                                                                     key=lambda kv: int(kv[0][0]))]


def num(m, k):
    return float(m[k]["value"].replace(",", ""))


def main(argv):
    rnd = argv[0]
    rest = argv[1:]
    tpath = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    os.makedirs(PROF, exist_ok=True)
    for i in range(0, len(rest), 3):
        cfg, prec, points = rest[i], rest[i + 1], int(rest[i + 2])
        rep = os.path.join(OUT, f"prof_{cfg}_{prec}.ncu-rep")
        metrics, stalls = raw(rep)
        launch = launches(os.path.join(OUT, f"launches_{cfg}_{prec}.csv"))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = num(metrics, "dram__bytes_read.sum") * scale[metrics["dram__bytes_read.sum"]["unit"]]
        wr = num(metrics, "dram__bytes_write.sum") * scale[metrics["dram__bytes_write.sum"]["unit"]]
        summary = {
            "round": rnd, "config": cfg, "prec": prec, "points": points,
            "capture": "ncu --set full --clock-control none --import-source on -k "
                       "regex:pointwise_kernel -s 3 -c 1 (bench.py --steps 5 --warmup 3 --n "
                       f"{points})",
            "dram_bytes_per_launch": rd + wr,
            "dram_bytes_per_point": (rd + wr) / points,
            "metrics": metrics, "stall_samples": stalls,
            "launch_list": launch,
        }
        with open(os.path.join(PROF, f"{rnd}_{cfg}_{prec}.json"), "w") as f:
            json.dump(summary, f, indent=1)
        traffic[f"{cfg}_{prec}"] = {"dram_bytes": rd + wr, "points": points,
                                    "source": f"profiles/{rnd}_{cfg}_{prec}.json"}
        print(f"{cfg} {prec}: {(rd + wr) / points:.1f} DRAM B/pt, "
              f"{metrics['gpu__time_duration.sum']['value']} {metrics['gpu__time_duration.sum']['unit']}, "
              f"dram {metrics['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']['value']}%, "
              f"top stalls {list(stalls.items())[:3]}")
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
