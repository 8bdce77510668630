"""Per-kernel summary of an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`).
python scripts/launch_summary.py gpurun_out/launches.csv"""
import collections
import csv
import sys


def main():
    lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = (r["Kernel Name"], r["Grid Size"])
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + float(r["Metric Value"]) / 1e3)
    tot = sum(t for _, t in agg.values())
    for (name, grid), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:5d} launches  {t / n:10.1f} us avg  {100 * t / tot:5.1f}% of GPU time  "
              f"{name[:60]} grid {grid}")


if __name__ == "__main__":
    main()
