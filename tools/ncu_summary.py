"""Summarise an ncu report: key throughput metrics + warp-stall breakdown.
usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, unit = rows[0], rows[1]
for vals in rows[2:]:
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print("kernel:", name[:100])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed.avg.per_cycle_elapsed", "smsp__inst_executed.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            print(f"  {k} = {vals[i]} {unit[i]}")
    tens = [(h, vals[i]) for i, h in enumerate(hdr) if "pipe_tensor" in h and h.endswith("pct_of_peak_sustained_active")]
    for h, v in tens[:6]:
        print(f"  {h} = {v}")
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls.append((float(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1.0
    print("  stall samples (share):", ", ".join(f"{n} {v / tot:.1%}" for v, n in sorted(stalls, reverse=True)[:8]))
