"""Extract the judged metrics of an ncu --set full capture into a small CSV
(kernel, metric, unit, value).  Usage: ncu_summary.py report.ncu-rep out.csv"""
import csv, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size"]
STALLS = "smsp__average_warps_issue_stalled_"

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout.splitlines()
rows = list(csv.reader(raw))
h, units = rows[0], rows[1]
with open(sys.argv[2], "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["kernel", "metric", "unit", "value"])
    for v in rows[2:]:
        d = dict(zip(h, v))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        for k in h:
            if k in KEYS or (k.startswith(STALLS) and k.endswith("_per_issue_active.ratio")):
                if d[k] not in ("", "0", "0.000000"):
                    w.writerow([name, k, units[h.index(k)], d[k]])
