"""Summarise ncu --set full reports of the decode kernel (the lines kept under
profiles/).  Usage: python tools/ncu_summary.py report.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active",
    "launch__grid_size",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum",
]
STALL = "smsp__average_warps_issue_stalled_"


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        val = dict(zip(head, row))
        unit = dict(zip(head, units))
        out.append(f"== {path.split('/')[-1]} {val.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in val:
                out.append(f"  {k} = {val[k]} {unit.get(k, '')}".rstrip())
        stalls = {}
        for k, v in val.items():
            if k.startswith(STALL) and k.endswith("_per_issue_active.ratio"):
                name = k[len(STALL):-len("_per_issue_active.ratio")]
                try:
                    stalls[name] = float(v)
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        out.append("  stalls: " + ", ".join(f"{k}:{100 * v / tot:.0f}%" for k, v in top))
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarise(p))
