# Round 2, call d: variants of the C4 step on the natural-order engine (device time).
set -x
mkdir -p gpurun_out
B='python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-time-to-tol'
$B > gpurun_out/r02d_default.json 2>&1
GSK_ARNOLDI=fused $B > gpurun_out/r02d_arnoldi_fused.json 2>&1
$B --schedule fused > gpurun_out/r02d_bicg_fused.json 2>&1
GSK_WPC=4 $B > gpurun_out/r02d_wpc4.json 2>&1
GSK_WPC=16 $B > gpurun_out/r02d_wpc16.json 2>&1
GSK_CARVEOUT=-1 $B > gpurun_out/r02d_carve_default.json 2>&1
GSK_CARVEOUT=50 $B > gpurun_out/r02d_carve50.json 2>&1
for f in gpurun_out/r02d_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), "gmres",
          round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
