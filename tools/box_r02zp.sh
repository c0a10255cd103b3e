# Round 2, call zp: fewer divergent branches in the stencil-slot row code (GSK_RCD_NB) — parity, A/B.
set -x
mkdir -p gpurun_out
GSK_LIB=$PWD/abvar/libgsk_nb1.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "row_classes or class_slots" 2>&1 | tail -2
for v in nb0 nb1 nb0b nb1b; do
  case $v in nb0|nb0b) unset GSK_LIB;; *) export GSK_LIB=$PWD/abvar/libgsk_nb1.so;; esac
  for cfg in C4 C3; do
    python bench.py --config $cfg --no-e2e --no-cpu --no-time-to-tol --no-plain-compare > gpurun_out/r02zp_${cfg}_$v.json 2> gpurun_out/r02zp_${cfg}_$v.err
  done
done
unset GSK_LIB
for f in gpurun_out/r02zp_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), "gmres", round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v}, d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
