# Round 2, call zi: SellView back to 128 bytes (row-class data behind one pointer) — parity, plain vs classes.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "row_classes or class_slots or spmv" > gpurun_out/r02zi_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r02zi_tests.log
for si in classes plain; do
  for cfg in C4 C3; do
    python bench.py --config $cfg --sell-index $si --no-e2e --no-cpu --no-time-to-tol --no-plain-compare > gpurun_out/r02zi_${cfg}_$si.json 2> gpurun_out/r02zi_${cfg}_$si.err
  done
done
for f in gpurun_out/r02zi_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "gmres", round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v}, d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
