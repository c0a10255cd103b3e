"""DRAM traffic per launch from an ncu --set full report -> profiles/<out>.json (read by
bench.py's roofline `traffic`).  Per kernel (short name, e.g. pass_kernel<2,1,OpS1>)
the launch with the most DRAM bytes is kept (early-exit launches of finished solves
move ~0 bytes).

    python tools/ncu_traffic.py report.ncu-rep profiles/r01_ncu_traffic.json "<source note>"
"""
import csv
import json
import re
import subprocess
import sys


def short(name):
    m = re.match(r"(?:void )?(?:gsk::)?(\w+)<(.*)>\(", name)
    if not m:
        return name.split("(")[0]
    args = [re.sub(r"gsk::|<.*?>", "", a).strip() for a in m.group(2).split(",")]
    return f"{m.group(1)}<{','.join(args)}>"


def main(rep, out, note):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    idx = {k: i for i, k in enumerate(rows[0])}
    units = rows[1]
    scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "B": 1e-9, "KB": 1e-6, "MB": 1e-3, "GB": 1.0}
    tscale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    kern = {}
    for r in rows[2:]:
        nm = short(r[idx["Kernel Name"]])
        rd = float(r[idx["dram__bytes_read.sum"]]) * scale[units[idx["dram__bytes_read.sum"]]]
        wr = float(r[idx["dram__bytes_write.sum"]]) * scale[units[idx["dram__bytes_write.sum"]]]
        us = float(r[idx["gpu__time_duration.sum"]]) * tscale[units[idx["gpu__time_duration.sum"]]]
        tot = (rd + wr) * 1e9
        if nm not in kern or tot > kern[nm]["bytes_per_launch"]:
            kern[nm] = {"dram_read_GB": round(rd, 6), "dram_write_GB": round(wr, 6), "us": us,
                        "bytes_per_launch": tot}
    with open(out, "w") as f:
        json.dump({"source": note, "kernels": kern}, f, indent=1)
    for k, v in kern.items():
        print(f"{k:40s} {v['bytes_per_launch'] / 1e9:8.3f} GB {v['us']:9.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
