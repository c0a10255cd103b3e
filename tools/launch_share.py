"""Per-kernel time shares of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_share.py launches.csv [more.csv ...]
"""
import collections
import csv
import re
import sys


def short(name):
    m = re.match(r"(?:void )?(?:gsk::)?(\w+)<(.*)>\(", name)
    if not m:
        return name.split("(")[0]
    args = [re.sub(r"gsk::|<.*?>", "", a).strip() for a in m.group(2).split(",")]
    return f"{m.group(1)}<{', '.join(args)}>"


def main(paths):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for p in paths:
        rows = [r for r in csv.reader(open(p)) if len(r) > 10]
        idx = {k: i for i, k in enumerate(rows[0])}
        for r in rows[1:]:
            if r[idx["Metric Name"]] != "gpu__time_duration.sum":
                continue
            v = float(r[idx["Metric Value"]])
            u = r[idx["Metric Unit"]]
            v *= {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}[u]
            k = short(r[idx["Kernel Name"]])
            tot[k] += v
            cnt[k] += 1
    s = sum(tot.values())
    print(f"{'kernel':42s} {'count':>6s} {'total_ns':>14s} {'mean_us':>9s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k:42s} {cnt[k]:6d} {v:14.1f} {v / cnt[k] / 1e3:9.1f} {100 * v / s:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1:])
