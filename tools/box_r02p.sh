# Round 2, call p: every graded run to its verdict vs the oracle (28 runs), then the full GPU suite.
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1 PYTHONFAULTHANDLER=1
timeout 1500 python tools/full_parity.py gpurun_out/r02_full_parity.json > gpurun_out/r02p_full_parity.log 2>&1; echo "full_parity rc=$?"
tail -6 gpurun_out/r02p_full_parity.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=10 > gpurun_out/r02p_gpu_tests.log 2>&1; echo "suite rc=$?"
tail -15 gpurun_out/r02p_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02p_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02p_smoke.log
