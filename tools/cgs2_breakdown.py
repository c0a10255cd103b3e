"""Per-step pass times of one CGS2 GMRES(30) cycle from an ncu launch list
(tools/prof_gmres_cycle.py under `ncu --metrics gpu__time_duration.sum --csv`)."""
import csv
import sys

N = 16777216
NNZ = 117047296
BA = 12 * NNZ + 4 * (N + 1)


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    idx = {k: i for i, k in enumerate(rows[0])}
    seq = []
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[idx["Metric Value"]])
        unit = r[idx["Metric Unit"]]
        v = v / 1e3 if unit == "nsecond" else (v * 1e3 if unit == "msecond" else v)  # -> us
        seq.append((r[idx["Kernel Name"]], v))
    j = 0
    tot = {"A": 0.0, "B": 0.0, "C": 0.0, "finish": 0.0}
    A = B = 0.0
    for nm, v in seq:
        if "mdot_pass<2" in nm or "mdot_pass<1" in nm:
            j += 1
            if j > 30:
                break
            A = v
            tot["A"] += v
        elif "mdot_pass<0" in nm and j:
            B = v
            tot["B"] += v
        elif "OpCgsC" in nm and "pass_kernel" in nm and j:
            tot["C"] += v
            gA = (BA + (j + 2) * 8 * N) / (A * 1e3)
            gB = ((2 * j + 2) * 8 * N) / (B * 1e3)
            gC = ((j + 2) * 8 * N) / (v * 1e3)
            print(f"j={j:2d}  A {A:7.1f} us {gA:5.2f} TB/s   B {B:7.1f} us {gB:5.2f} TB/s (2j+2 vectors)   "
                  f"C {v:7.1f} us {gC:5.2f} TB/s")
        elif "finish" in nm and j:
            tot["finish"] += v
    print({k: round(v / 1e3, 2) for k, v in tot.items()}, "ms per cycle")


if __name__ == "__main__":
    main(sys.argv[1])
