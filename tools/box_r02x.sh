set -x
mkdir -p gpurun_out
python tools/e2e_breakdown.py C4 > gpurun_out/r02x_e2e.log 2>&1; cat gpurun_out/r02x_e2e.log
