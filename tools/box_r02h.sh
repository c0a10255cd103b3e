# Round 2, call h: full GPU suite on the v13 engine (natural windows + L2 prefetch),
# the default bench line, a wpc16 variant, and the per-config table.
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/r02h_gpu_tests.log 2>&1; echo "suite rc=$?"
tail -20 gpurun_out/r02h_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; echo "bench rc=$?"
GSK_WPC=16 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-time-to-tol > gpurun_out/r02h_wpc16.json 2>&1
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-time-to-tol > gpurun_out/r02h_default_short.json 2>&1
timeout 1500 python tools/run_configs.py gpurun_out/r02_configs > gpurun_out/r02h_configs.log 2>&1; echo "configs rc=$?"
for f in gpurun_out/r02h_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "gmres",
          round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
