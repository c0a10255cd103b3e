# Round 2, call zm: row-class passes reducing the leaves of 2 / 4 windows together — parity, A/B.
set -x
mkdir -p gpurun_out
for v in lb4 lb2; do
  GSK_LIB=$PWD/abvar/libgsk_$v.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "row_classes or class_slots" > gpurun_out/r02zm_tests_$v.log 2>&1; echo "tests $v rc=$?"
  tail -2 gpurun_out/r02zm_tests_$v.log
done
for v in lb1 lb2 lb4; do
  if [ $v = lb1 ]; then unset GSK_LIB; else export GSK_LIB=$PWD/abvar/libgsk_$v.so; fi
  for cfg in C4 C3; do
    python bench.py --config $cfg --no-e2e --no-cpu --no-time-to-tol --no-plain-compare > gpurun_out/r02zm_${cfg}_$v.json 2> gpurun_out/r02zm_${cfg}_$v.err
  done
done
unset GSK_LIB
for f in gpurun_out/r02zm_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "gmres", round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v}, d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
