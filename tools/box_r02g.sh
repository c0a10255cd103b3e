# Round 2, call g: TMA L2 bulk prefetch of upcoming windows (GSK_L2PF), plain SELL and SELL-U.
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "uniform" > gpurun_out/r02g_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02g_tests.log
GSK_L2PF=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "uniform or test_bicgstab_parity" > gpurun_out/r02g_tests_pf.log 2>&1; echo "tests pf rc=$?"
tail -3 gpurun_out/r02g_tests_pf.log
B='python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-time-to-tol'
for pf in 0 1 2; do
  GSK_L2PF=$pf $B > gpurun_out/r02g_plain_pf$pf.json 2>&1
  GSK_L2PF=$pf $B --sell-index uniform > gpurun_out/r02g_sellu_pf$pf.json 2>&1
done
for f in gpurun_out/r02g_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "gmres",
          round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
