# Round 2, call ze: default bench line with the row-class dictionary (roofline on the kernel with the largest share), then the full GPU suite.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r02ze_bench.json 2> gpurun_out/r02ze_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r02ze_bench.err
python - <<'PY'
import json
d = json.loads(open('gpurun_out/r02ze_bench.json').read().strip().splitlines()[-1]); x = d["extra"]
print(d["value"], d["ms_per_step"], d["e2e"], d["clocks"])
print({k: (round(v, 4) if isinstance(v, float) else v) for k, v in d["roofline"].items()})
for r in x["roofline_all"]:
    print("   ", r["kernel"][:40], round(r["ms_per_launch"], 4), round(r["frac"], 3), round(r["share_of_step"], 3), r["traffic"])
print(x["bicgstab"]["iters_per_s"], x["gmres"]["iters_per_s"], x["spmv"], x["sell_plain"])
print(x["time_to_tol"])
print(d["config"]["format"]); print(d["config"]["l2"]); print(d["cpu_baseline"])
PY
timeout 3000 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02ze_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r02ze_tests.log
