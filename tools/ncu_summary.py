#!/usr/bin/env python
"""One-page summary of an ncu --set full capture of the fused kernel (reads the
.ncu-rep with `ncu -i ... --page raw --csv`)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "fp64 datapath (shared pipe) busy %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA subpipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "DFMA-class fp64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__occupancy_limit_registers", "CTA limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1/smem LSU wavefronts %"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math pipe / issue"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[2]
    d = {name: (val, unit) for name, unit, val in zip(h, u, v)}
    print(f"kernel: {d.get('Kernel Name', ('?',))[0]}  grid {d.get('Grid Size', ('?',))[0]} block {d.get('Block Size', ('?',))[0]}")
    for k, label in KEYS:
        if k in d:
            print(f"  {label:38s} {d[k][0]:>16s} {d[k][1]}")


if __name__ == "__main__":
    main(sys.argv[1])
