"""Markdown summary of one kernel from an `ncu --set full` report: time,
launch shape, pipe utilisation (DMMA / FP64 / LSU), DRAM traffic, L2 hit
rate, shared-memory wavefronts and bank conflicts, warp stall reasons.

    python tools/ncu_summary.py gpurun_out/r02/gather_tc_c5.ncu-rep > profiles/r02/gather_tc_m6_c5.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", 1e-6, "ms"),
    ("sm__cycles_elapsed.avg.per_second", 1e-9, "GHz"),
    ("launch__grid_size", 1, ""),
    ("launch__block_size", 1, ""),
    ("launch__registers_per_thread", 1, "register/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", 1, "%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1, "%"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 1, "%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1, "%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1, "%"),
    ("dram__bytes_read.sum", 1e-9, "GB"),
    ("dram__bytes_write.sum", 1e-9, "GB"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1, "%"),
    ("lts__t_sector_hit_rate.pct", 1, "%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1, ""),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1, ""),
    ("smsp__inst_executed.sum", 1, "inst"),
    ("smsp__inst_executed_pipe_fp64.sum", 1, "inst"),
]


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    name = d.get("Kernel Name", "?")
    print(f"## {name}\n\nSource: `{rep}` (ncu --set full --clock-control none, one launch)\n")
    print("| metric | value | unit |\n|---|---|---|")
    for k, _, _ in METRICS:
        if k in d and d[k] not in ("", "n/a"):
            print(f"| {k} | {d[k]} | {u.get(k, '')} |")
    stalls = []
    for k, val in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(val.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("\nWarp stall reasons (cycles per issued instruction):\n")
    for val, k in sorted(stalls, reverse=True)[:10]:
        if val > 0.05:
            print(f"- {k}: {val:.3f}")


if __name__ == "__main__":
    main()
