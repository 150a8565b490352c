"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``) per kernel.

  python tools/ncu_summary.py gpurun_out/launches_emr.csv > profiles/r01_launches_emr.txt

ncu serialises launches and runs them cold-cache, so compare the SHARES with the live
per-kernel shares bench.py prints, not the absolute times (B200_PROFILING.md).
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path):
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        us = float(r["Metric Value"].replace(",", "")) * SCALE[r["Metric Unit"]]
        a = agg.setdefault(name, [0, 0.0, r["Grid Size"], r["Block Size"]])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"# {path}: {sum(a[0] for a in agg.values())} launches, {tot:.1f} us total")
    print(f"{'kernel':<48} {'launches':>8} {'total_us':>11} {'us/launch':>10} {'share':>6}  grid x block")
    for name, (n, us, grid, block) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:48]:<48} {n:>8} {us:>11.1f} {us / n:>10.2f} {us / tot:>6.3f}  {grid} x {block}")


if __name__ == "__main__":
    main(sys.argv[1])
