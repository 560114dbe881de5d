"""Summarise an `ncu --set full` report of one bench frame into profiles/.

    python tools/ncu_summary.py gpurun_out/m_full.ncu-rep profiles/r1_ncu_full_summary.json \
        profiles/ncu_traffic.json hd4

Writes the per-kernel metric subset (the first JSON) and the insert kernel's DRAM
traffic, instruction and RED-sector counts that bench.py's roofline objects read (the
second JSON).
"""

import csv
import io
import json
import subprocess
import sys

METRICS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
           "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum")
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, out_summary, out_traffic, workload="hd4"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    summary, traffic = [], {}
    for r in rows[2:]:
        k = {"Kernel Name": r[head.index("Kernel Name")]}
        for m in METRICS:
            if m in head:
                i = head.index(m)
                k[m] = f"{r[i]} {units[i]}".strip()
        summary.append(k)
        if "insert_frame_kernel" in k["Kernel Name"]:
            def val(m):
                i = head.index(m)
                return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
            traffic = {
                "insert_frame_kernel": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                "_source": f"{out_summary} ({rep}: ncu --set full of one bench.py frame after 3 "
                           "warm-up frames, traced App. B stream): per-launch "
                           "dram__bytes_read.sum + dram__bytes_write.sum, smsp__inst_executed.sum, "
                           "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum of "
                           "insert_frame_kernel",
                "insert_frame_kernel_inst": val("smsp__inst_executed.sum"),
                "insert_frame_kernel_red_sectors":
                    val("l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum"),
            }
    json.dump(summary, open(out_summary, "w"), indent=1)
    try:
        merged = json.load(open(out_traffic))
    except (OSError, ValueError):
        merged = {}
    if traffic:
        merged[workload] = traffic  # keyed by bench workload (bench.py _traffic)
    json.dump(merged, open(out_traffic, "w"), indent=1)
    for k in summary:
        print(k["Kernel Name"][:40], k.get("gpu__time_duration.sum"), k.get("smsp__inst_executed.sum"))


if __name__ == "__main__":
    main(*sys.argv[1:5])
