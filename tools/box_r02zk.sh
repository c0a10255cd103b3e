# Round 2, call zk: windows per CTA of the row-class passes (GSK_WPC) with the CTA-level prefetch, C4 / C3.
set -x
mkdir -p gpurun_out
for w in 4 8 16; do
  for cfg in C4 C3; do
    GSK_WPC=$w python bench.py --config $cfg --no-e2e --no-cpu --no-time-to-tol --no-plain-compare > gpurun_out/r02zk_${cfg}_w$w.json 2> gpurun_out/r02zk_${cfg}_w$w.err
  done
done
for f in gpurun_out/r02zk_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "gmres", round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v}, d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
