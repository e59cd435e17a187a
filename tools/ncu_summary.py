"""Key metrics per kernel from an ncu report: python tools/ncu_summary.py rep.ncu-rep [name-filter]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA pipe % (active)"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem->TC % (elapsed)"),
    ("sm__cycles_active.avg", "sm active cyc"),
    ("sm__cycles_elapsed.avg", "elapsed cyc"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "st math"),
    ("smsp__pcsamp_warps_issue_stalled_wait", "st wait"),
    ("smsp__pcsamp_warps_issue_stalled_barrier", "st barrier"),
    ("smsp__pcsamp_warps_issue_stalled_long_scoreboard", "st long_sb"),
    ("smsp__pcsamp_warps_issue_stalled_short_scoreboard", "st short_sb"),
    ("smsp__pcsamp_warps_issue_stalled_mio_throttle", "st mio"),
    ("smsp__pcsamp_warps_issue_stalled_lg_throttle", "st lg"),
    ("smsp__pcsamp_warps_issue_stalled_not_selected", "st not_sel"),
    ("smsp__pcsamp_warps_issue_stalled_selected", "selected"),
    ("smsp__pcsamp_warps_issue_stalled_dispatch_stall", "st dispatch"),
    ("smsp__pcsamp_warps_issue_stalled_no_instructions", "st no_inst"),
    ("smsp__pcsamp_warps_issue_stalled_membar", "st membar"),
    ("smsp__pcsamp_warps_issue_stalled_branch_resolving", "st branch"),
    ("smsp__pcsamp_warps_issue_stalled_imc_miss", "st imc"),
]

rep = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "")
    if flt not in name:
        continue
    print(name.replace("(anonymous namespace)::", "")[:90], d.get("Grid Size"))
    print("   " + "  ".join(f"{lab}={d[k]}" for k, lab in KEYS if k in d))
