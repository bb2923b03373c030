"""Print the key ncu metrics of every kernel in an .ncu-rep (run here, no GPU)."""
import csv
import subprocess
import sys

KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "L2 Cache Throughput"),
    ("GPU Speed Of Light Throughput", "L1/TEX Cache Throughput"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("Memory Workload Analysis", "Memory Throughput"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Memory Workload Analysis", "L1/TEX Hit Rate"),
    ("Occupancy", "Achieved Active Warps Per SM"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
    ("Scheduler Statistics", "Issued Warp Per Scheduler"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki, si, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Section Name", "Metric Name", "Metric Value",
                                                      "Metric Unit", "ID"))
    by = {}
    for r in rows[1:]:
        by.setdefault((r[ii], r[ki]), {})[(r[si], r[mi])] = (r[vi], r[ui])
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    rh = rr[0]
    dr = [rh.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum")]
    units = rr[1]
    for n, ((kid, kname), m) in enumerate(by.items()):
        print(f"--- [{kid}] {kname[:100]}")
        for k in KEYS:
            if k in m:
                print(f"    {k[1]:40s} {m[k][0]} {m[k][1]}")
        row = rr[2 + n]
        print(f"    {'dram read / write':40s} {row[dr[0]]} {units[dr[0]]} / {row[dr[1]]} {units[dr[1]]}")


if __name__ == "__main__":
    main(sys.argv[1])
