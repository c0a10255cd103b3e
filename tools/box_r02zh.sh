# Round 2, call zh: Bi-CGSTAB schedules on row-class plans (split / split4 / fused), C4 and C3.
set -x
mkdir -p gpurun_out
for sc in split split4 fused; do
  for cfg in C4 C3; do
    python bench.py --config $cfg --schedule $sc --no-e2e --no-cpu --no-time-to-tol --no-plain-compare > gpurun_out/r02zh_${cfg}_$sc.json 2> gpurun_out/r02zh_${cfg}_$sc.err
  done
done
for f in gpurun_out/r02zh_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "gmres", round(x["gmres"]["iters_per_s"], 1), {k: round(v, 4) for k, v in x["probe_ms"].items() if v}, d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
