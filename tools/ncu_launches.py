"""Condense an ncu --csv launch list (gpu__time_duration.sum per launch) into id,kernel,grid,block,ns.

    python tools/ncu_launches.py gpurun_out/launches_c1.csv "<command>" > profiles/<name>.csv
"""
import csv
import sys


def main(path, cmd):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, gi, bi = hdr.index("Kernel Name"), hdr.index("Grid Size"), hdr.index("Block Size")
    mi, vi, ii, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID"), hdr.index("Metric Unit")
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none: {cmd}")
    print("# (cold-cache, serialised; compare shares, not absolutes)")
    print("id,kernel,grid,block,gpu__time_duration_ns")
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r[ui], 1)
        name = r[ki].split("(")[0]
        print(f'{r[ii]},"{name}","{r[gi]}","{r[bi]}",{int(v * scale)}')


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
