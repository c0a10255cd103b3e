# Round 2, call f: SELL-U (chunk-uniform column deltas) — parity, then the C4 step.
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "uniform or sell_layout or sell_dict" > gpurun_out/r02f_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02f_tests.log
B='python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-time-to-tol'
$B --sell-index uniform > gpurun_out/r02f_sellu.json 2>&1
GSK_WPC=16 $B --sell-index uniform > gpurun_out/r02f_sellu_wpc16.json 2>&1
$B > gpurun_out/r02f_plain.json 2>&1
for f in gpurun_out/r02f_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "gmres",
          round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
