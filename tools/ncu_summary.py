"""Summarise an ncu report (raw page) per kernel: time, DRAM bytes, throughputs."""
import csv
import re
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size"]
SHORT = ["us", "dramR_GB", "dramW_MB", "dram%", "l1%", "l2%", "l2hit%", "warps%", "regs", "grid"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    idx = {k: i for i, k in enumerate(rows[0])}
    print("kernel".ljust(22), " ".join(s.rjust(9) for s in SHORT))
    for row in rows[2:]:
        name = row[idx["Kernel Name"]]
        m = re.search(r"(?:fused|stream)_pass<(\d), gsk::(\w+)>", name)
        nm = f"{m.group(1)} {m.group(2)}" if m else name.split("(")[0][-22:]
        print(nm.ljust(22), " ".join(row[idx[c]][:9].rjust(9) if c in idx else "-".rjust(9) for c in WANT))


if __name__ == "__main__":
    main(sys.argv[1])
