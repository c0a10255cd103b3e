# Round 2, call zo: CTAs per SM of the row-class passes again, now with the CTA-level prefetch and 16 windows per CTA.
set -x
mkdir -p gpurun_out
for v in m4 m5 m6; do
  if [ $v = m4 ]; then unset GSK_LIB; else export GSK_LIB=$PWD/abvar/libgsk_$v.so; fi
  for cfg in C4 C3; do
    python bench.py --config $cfg --no-e2e --no-cpu --no-time-to-tol --no-plain-compare > gpurun_out/r02zo_${cfg}_$v.json 2> gpurun_out/r02zo_${cfg}_$v.err
  done
done
unset GSK_LIB
for f in gpurun_out/r02zo_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), "gmres", round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v}, d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
