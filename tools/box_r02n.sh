# Round 2, call n: windows per CTA x L2 prefetch on C3 / C5 (C4 reference), and the fault hook parity.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fault or peer" > gpurun_out/r02n_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02n_tests.log
for cfg in C3 C5; do
  for w in 2 4 8; do
    for pf in 0 1; do
      GSK_WPC=$w GSK_L2PF=$pf python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-time-to-tol > gpurun_out/r02n_${cfg}_w${w}_pf${pf}.json 2>&1
    done
  done
done
for f in gpurun_out/r02n_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), "gmres",
          round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
