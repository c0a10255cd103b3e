# Round 2, call k: full-size parity vs the oracle records present (C1-C5).
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1
timeout 1500 python tools/full_parity.py gpurun_out/r02_full_parity.json > gpurun_out/r02k_full_parity.log 2>&1; echo "full_parity rc=$?"
tail -40 gpurun_out/r02k_full_parity.log
