# Round 2, call t: coop v2 with parallel flag polling; register budget 2/3/4 CTAs per SM.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "coop" > gpurun_out/r02u_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02u_tests.log
for mb in 2 3; do
GSK_COOP_MINB=$mb timeout 600 python tools/coop_timing.py gpurun_out/r02u_coop_m$mb.json --cases=C2:200,C2:256,C2:None,C3:64,C5:512,C2:724 > gpurun_out/r02u_coop_m$mb.log 2>&1
python - gpurun_out/r02u_coop_m$mb.json <<'PY'
import json,sys
for r in json.load(open(sys.argv[1])): print(sys.argv[1][-8:], r["config"], r["n"], r["bit_identical"], round(r["us_per_it_graph"],1), round(r["us_per_it_coop"],1))
PY
done
