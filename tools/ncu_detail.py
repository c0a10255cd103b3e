"""Per-kernel detail from an ncu --set full report (run on the GPU box; the raw report
is too large to bring back): for the heaviest launch of each kernel, time, DRAM bytes,
DRAM / L2 / L1 throughput, L2 sectors and hit rate, L1 hit rate, registers, occupancy
and the top warp-stall reasons (cycles per issued instruction).

    python tools/ncu_detail.py report.ncu-rep out.json "<what was captured>"
"""
import csv
import json
import re
import subprocess
import sys

METRICS = {
    "us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_sectors": "lts__t_sectors.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
STALL = re.compile(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$")


def short(name):
    m = re.match(r"(?:void )?(?:gsk::)?(\w+)<(.*)>\(", name)
    if not m:
        return name.split("(")[0]
    args = [re.sub(r"gsk::|<.*?>", "", a).strip() for a in m.group(2).split(",")]
    return f"{m.group(1)}<{','.join(args)}>"


def num(row, idx, units, key):
    if key not in idx:
        return None
    try:
        v = float(row[idx[key]].replace(",", ""))
    except ValueError:
        return None
    return v * SCALE.get(units[idx[key]], 1.0)


def main(rep, out, note):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    idx = {k: i for i, k in enumerate(rows[0])}
    units = rows[1]
    stall_cols = [(m.group(1), k) for k in idx for m in [STALL.match(k)] if m]
    kern = {}
    for r in rows[2:]:
        nm = short(r[idx["Kernel Name"]])
        d = {k: num(r, idx, units, v) for k, v in METRICS.items()}
        d["dram_bytes"] = (d["dram_read"] or 0) + (d["dram_write"] or 0)
        stalls = {s: num(r, idx, units, k) for s, k in stall_cols}
        d["top_stalls"] = dict(sorted(((s, round(v, 2)) for s, v in stalls.items() if v), key=lambda t: -t[1])[:5])
        if nm not in kern or d["dram_bytes"] > kern[nm]["dram_bytes"]:
            kern[nm] = d
    with open(out, "w") as f:
        json.dump({"source": note, "kernels": kern}, f, indent=1)
    for nm, d in kern.items():
        print(f"{nm[:40]:40s} {d['us']:9.1f} us  DRAM {d['dram_bytes'] / 1e9:7.3f} GB {d['dram_pct'] or 0:5.1f}%  "
              f"L2 {d['l2_pct'] or 0:5.1f}% hit {d['l2_hit_pct'] or 0:5.1f}%  L1 hit {d['l1_hit_pct'] or 0:5.1f}%  "
              f"{d['top_stalls']}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
