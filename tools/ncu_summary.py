"""Selected metrics + warp-stall samples of every kernel in an ncu report, as csv rows
(kernel, launch, metric, unit, value).   python tools/ncu_summary.py X.ncu-rep > out.csv"""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_shared_mem"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
w = csv.writer(sys.stdout)
w.writerow(["kernel", "launch", "metric", "unit", "value"])
for li, v in enumerate(rows[2:]):
    name = v[h.index("Kernel Name")].split("(")[0]
    for x in WANT:
        if x in h:
            i = h.index(x)
            w.writerow([name, li, x, u[i], v[i]])
    for i, x in enumerate(h):
        if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued") and v[i] not in ("0", ""):
            w.writerow([name, li, x, u[i], v[i]])
