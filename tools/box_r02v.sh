# Round 2, call v: scatter/gather probe at C5 size; coop AUTO range.
set -x
mkdir -p gpurun_out
python tools/scatter_probe.py > gpurun_out/r02v_scatter.log 2>&1; cat gpurun_out/r02v_scatter.log
GSK_COOP_MINB=2 timeout 600 python tools/coop_timing.py gpurun_out/r02v_coop.json --cases=C2:160,C2:200,C2:256,C2:300,C2:362,C3:40,C3:48,C5:200,C5:256,C5:362 > gpurun_out/r02v_coop.log 2>&1
python - gpurun_out/r02v_coop.json <<'PY'
import json,sys
for r in json.load(open(sys.argv[1])): print(r["config"], r["n"], r["bit_identical"], round(r["us_per_it_graph"],1), round(r["us_per_it_coop"],1))
PY
