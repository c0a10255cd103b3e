# Round 2, call e: SELL-D (uint8 column index) on the natural-order engine vs plain SELL.
set -x
mkdir -p gpurun_out
B='python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-time-to-tol'
$B --sell-index dict > gpurun_out/r02e_selld.json 2>&1
GSK_WPC=16 $B > gpurun_out/r02e_wpc16.json 2>&1
for f in gpurun_out/r02e_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), "gmres",
          round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
