"""One-line-per-metric brief of every kernel in an ncu --set full report
(duration, DRAM bytes/throughput, SM/L1 throughput, issue, occupancy, pipe
utilisation), for profiles/*.md."""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]
want = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
        ("dram__bytes_write.sum", "dram write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
        ("launch__registers_per_thread", "registers/thread"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
        ("smsp__inst_executed.sum", "warp instructions")]
ki = h.index("Kernel Name")
for r in data:
    name = r[ki].split("(")[0].replace("void ", "")
    print(f"\n### {name}  (grid {r[h.index('Grid Size')]}, block {r[h.index('Block Size')]})")
    for key, label in want:
        if key in h:
            i = h.index(key)
            print(f"- {label}: {r[i]} {units[i]}")
