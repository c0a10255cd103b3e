# Round 2, call q: four-pass Bi-CGSTAB schedule (S0 folded into S4/S1) — parity and speed.
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bicgstab_parity or fault" > gpurun_out/r02q_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02q_tests.log
for cfg in C2 C3 C4 C5; do
  for sc in split split4; do
    python bench.py --config $cfg --schedule $sc --steps 3 --warmup 3 --no-e2e --no-cpu --no-time-to-tol > gpurun_out/r02q_${cfg}_${sc}.json 2>&1
  done
done
for f in gpurun_out/r02q_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
