"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
total time, launch count and share per kernel (first 80 chars of the name).

    python tools/launch_summary.py gpurun_out/launches.csv [--skip N] [--md]
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--skip", type=int, default=0, help="ignore the first N launches (warm-up)")
    ap.add_argument("--md", action="store_true")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    data = [dict(zip(h, r)) for r in rows[start + 1:] if len(r) == len(h)]
    data = [d for d in data if d.get("Metric Name") == "gpu__time_duration.sum"][a.skip:]
    agg = collections.OrderedDict()
    for d in data:
        k = d["Kernel Name"][:80]
        agg.setdefault(k, [0, 0.0])
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(t for _, t in agg.values())
    if a.md:
        print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if a.md:
            print(f"| `{k}` | {n} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
        else:
            print(f"{t / 1e6:9.3f} ms {n:4d} {100 * t / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main()
