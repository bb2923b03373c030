"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into per-kernel shares.

    python scripts/summarize_launches.py gpurun_out/r01_launches.csv [--skip-setup]
"""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
        rows.append((int(r["ID"]), r["Kernel Name"], v * scale, r.get("Grid Size", ""), r.get("Block Size", "")))
    return rows


def main():
    path = sys.argv[1]
    rows = load(path)
    setup = {"sell_width_kernel", "sell_fill_kernel", "DeviceScanInitKernel", "DeviceScanKernel", "l1_dinv_kernel",
             "vectorized_elementwise_kernel", "elementwise_kernel"}
    body = [r for r in rows if r[1].split("(")[0].split("<")[0] not in setup]
    tot = sum(r[2] for r in body)
    agg = OrderedDict()
    for _, name, us, grid, blk in body:
        key = name.split("(")[0] + (f" g{grid}" if "--by-grid" in sys.argv else "")
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += us
    print(f"launches={len(body)} total_us={tot:.1f}")
    print(f"{'kernel':52s} {'n':>6s} {'total_us':>10s} {'avg_us':>9s} {'share':>7s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:52]:52s} {n:6d} {us:10.1f} {us / n:9.2f} {100 * us / tot:6.1f}%")


if __name__ == "__main__":
    main()
