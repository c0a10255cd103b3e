# Round 2, call zl: no stream-ordered allocations / pinned frees in the plan life cycle — shard tests, e2e stability, bench.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "shard or dot or concurrent or plans" > gpurun_out/r02zl_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02zl_tests.log
E2E_STEPS=24 python tools/e2e_breakdown.py C4 > gpurun_out/r02_e2e_breakdown_v18.txt 2>&1; cat gpurun_out/r02_e2e_breakdown_v18.txt
python bench.py > gpurun_out/r02zl_bench.json 2> gpurun_out/r02zl_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/r02zl_bench.json').read().strip().splitlines()[-1]); x = d["extra"]
print(d["value"], d["ms_per_step"], d["e2e"], d["clocks"])
for r in x["roofline_all"]:
    print("   ", r["kernel"][:40], round(r["ms_per_launch"], 4), round(r["frac"], 3), round(r["share_of_step"], 3), r["traffic"])
for k,v in x["time_to_tol"].items():
    for kk,vv in v.items(): print(k,kk,round(vv["ms"]),vv["iterations"],vv["status"])
print(x["sell_plain"])
PY
python bench.py --shards 8 --steps 2 --warmup 2 > gpurun_out/r02zl_shards8.json 2> gpurun_out/r02zl_shards8.err; python -c "
import json;d=json.loads(open('gpurun_out/r02zl_shards8.json').read().strip().splitlines()[-1]);print(8, d['value'], d['e2e'])"
