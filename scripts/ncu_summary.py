"""Summarise an ncu report: key metrics + stall reasons (usage: ncu_summary.py rep)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, vals = rows[0], rows[2]
d = dict(zip(hdr, vals))
def g(k):
    try:
        return float(d[k])
    except (KeyError, ValueError):
        return None
keys = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "sm_cycles": ("sm__cycles_elapsed.avg", 1),
    "inst_executed(warp)": ("smsp__inst_executed.sum", 1),
    "ipc_per_sm": ("sm__inst_executed.avg.per_cycle_active", 1),
    "issue_active_pct": ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", 1),
    "warps_active_per_sm": ("sm__warps_active.avg.per_cycle_active", 1),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "fp64_pipe_pct": ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "lsu_pipe_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    "dram_read_B": ("dram__bytes_read.sum", 1),
    "dram_write_B": ("dram__bytes_write.sum", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "regs": ("launch__registers_per_thread", 1),
    "smem_per_block_B": ("launch__shared_mem_per_block_dynamic", 1),
}
for name, (k, sc) in keys.items():
    v = g(k)
    print(f"{name:26s} {v * sc if v is not None else 'n/a'}")
stalls = [(g(k), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in hdr
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
stalls = [(v, k) for v, k in stalls if v]
tot = sum(v for v, _ in stalls)
print("stall reasons (pc sampling):")
for v, k in sorted(stalls, reverse=True)[:10]:
    print(f"  {v / tot * 100:5.1f}% {k}")
