"""Summarise ncu artefacts for profiles/: a full-set .ncu-rep (key metrics,
stall reasons, hottest SASS) or a --metrics gpu__time_duration launch list.

    python tools/ncu_summary.py rep  gpurun_out/x.ncu-rep  > profiles/r01/x.md
    python tools/ncu_summary.py list gpurun_out/launches.csv > profiles/r01/launches.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum",
]


def rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"## {name[:120]}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {k} | {r[i]} | {units[i]} |")
        stalls = []
        for i, k in enumerate(hdr):
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        print("\nWarp stall reasons (cycles per issued instruction):\n")
        for v, k in sorted(stalls, reverse=True)[:8]:
            print(f"- {k}: {v:.3f}")
        print()


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = {}
    order = []
    for r in rows[1:]:
        short = r[ik].split("(")[0].replace("void ", "")[:80]
        if short not in tot:
            order.append(short)
            tot[short] = [0, 0.0]
        tot[short][0] += 1
        tot[short][1] += float(r[iv].replace(",", ""))
    total = sum(v[1] for v in tot.values())
    print("| kernel | launches | total ns | share |\n|---|---|---|---|")
    for k in sorted(order, key=lambda k: -tot[k][1]):
        n, t = tot[k]
        print(f"| `{k}` | {n} | {t:.0f} | {t / total * 100:.1f}% |")


if __name__ == "__main__":
    {"rep": rep, "list": launches}[sys.argv[1]](sys.argv[2])
