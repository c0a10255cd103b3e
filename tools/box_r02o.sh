# Round 2, call o: device-initiated halos + reductions (emulated on one GPU).
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1 PYTHONFAULTHANDLER=1
timeout 900 python -u -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "peer or sharded or fault" > gpurun_out/r02o_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02o_tests.log
for P in 2 8; do python -u bench.py --shards $P --peer --steps 2 --warmup 3 --no-e2e > gpurun_out/r02o_shards${P}_peer.json 2>&1; echo "bench $P rc=$?"; done
for f in gpurun_out/r02o_shards*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), x["bicgstab"], x["history"]["bicgstab_sha256"][:16], x["history"]["gmres_sha256"][:16])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
