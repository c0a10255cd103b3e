# Round 2, call l: device-initiated shard reductions (emulated on one GPU) — parity and cost.
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_abi.py tests/test_multi_gpu.py -q -x -p no:cacheprovider -k "peer or sharded or layouts" > gpurun_out/r02l_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02l_tests.log
for P in 2 8; do
  python bench.py --shards $P --steps 2 --warmup 3 --no-e2e > gpurun_out/r02l_shards$P.json 2>&1
  python bench.py --shards $P --peer --steps 2 --warmup 3 --no-e2e > gpurun_out/r02l_shards${P}_peer.json 2>&1
done
for f in gpurun_out/r02l_shards*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), x["bicgstab"], x["history"], d["comm"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
