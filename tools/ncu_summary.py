"""Summarise .ncu-rep captures into a small text table for profiles/:
duration, IPC, issue-slot busy, occupancy, DRAM bytes (read+write), L2 hit
rate, pipe utilisation (ALU / FMA / XU / FP64 / LSU) and the top stall
reasons.

    python tools/ncu_summary.py out.txt a.ncu-rep [b.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        res.append((d, u))
    return res


def main():
    out = open(sys.argv[1], "w")
    for path in sys.argv[2:]:
        for d, u in raw(path):
            out.write(f"== {path}  kernel={d.get('Kernel Name', '?')[:80]}\n")
            for k in KEYS:
                if k in d:
                    out.write(f"  {k:62s} {d[k]:>18s} {u.get(k, '')}\n")
            stalls = sorted(((float(v.replace(',', '') or 0), k) for k, v in d.items()
                             if k.startswith("smsp__average_warp_latency_issue_stalled_")
                             or k.startswith("smsp__pcsamp_warps_issue_stalled_")
                             and not k.endswith("_not_issued")
                             if v.replace(',', '').replace('.', '').isdigit()), reverse=True)[:8]
            for v, k in stalls:
                out.write(f"  {k:62s} {v:>18.0f}\n")
    out.close()


if __name__ == "__main__":
    main()
