# Round 2, call j: short-slot kernels (<= 5 slots per lane, 5 CTAs/SM) on the 2-D configs;
# parity of the touched paths first.
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bicgstab_parity or gmres_parity or sell or full_c4 or sharded" > gpurun_out/r02j_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02j_tests.log
timeout 900 python -m pytest tests/test_full_parity.py -q -x -p no:cacheprovider -k "C2 or C1" > gpurun_out/r02j_full.log 2>&1; echo "full rc=$?"
tail -3 gpurun_out/r02j_full.log
for cfg in C2 C5 C4; do
  B="python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-time-to-tol"
  $B > gpurun_out/r02j_${cfg}_short.json 2>&1
  GSK_SHORT=0 $B > gpurun_out/r02j_${cfg}_noshort.json 2>&1
done
for f in gpurun_out/r02j_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "gmres",
          round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
