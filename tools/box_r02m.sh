# Round 2, call m: device-initiated reductions after the host/device fix; C4 GMRES full parity.
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1 PYTHONFAULTHANDLER=1 PYTHONUNBUFFERED=1
timeout 600 python -u -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "peer" > gpurun_out/r02m_peer.log 2>&1; echo "peer rc=$?"
tail -30 gpurun_out/r02m_peer.log
timeout 900 python -u -m pytest tests/test_gpu_parity.py tests/test_abi.py -q -x -p no:cacheprovider -k "sharded or layouts" > gpurun_out/r02m_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02m_tests.log
for P in 2 8; do python -u bench.py --shards $P --peer --steps 2 --warmup 3 --no-e2e > gpurun_out/r02m_shards${P}_peer.json 2>&1; echo "bench $P rc=$?"; tail -c 600 gpurun_out/r02m_shards${P}_peer.json; done
timeout 900 python -u -m pytest tests/test_full_parity.py -q -x -p no:cacheprovider -k "C4" > gpurun_out/r02m_full_c4.log 2>&1; echo "full c4 rc=$?"
tail -5 gpurun_out/r02m_full_c4.log
