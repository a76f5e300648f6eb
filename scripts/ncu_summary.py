"""Print the key ncu counters of every kernel in a .ncu-rep (raw page)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(f"## {d.get('Kernel Name', '?')[:120]}")
    for k in KEYS:
        if k in d:
            print(f"- {k} = {d[k]}")
    st = [(k, v) for k, v in d.items() if "smsp__pcsamp_warps_issue_stalled" in k
          and not k.endswith("not_issued")]
    st = sorted(st, key=lambda kv: -float(kv[1].replace(",", "") or 0))[:6]
    print("- top stall samples: " + ", ".join(f"{k.split('stalled_')[1]}={v}" for k, v in st))
    print()
