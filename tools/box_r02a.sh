# Round 2, first GPU call: GPU suite, full-size parity vs the oracle records present,
# the default bench line and its launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 -p no:cacheprovider > gpurun_out/r02a_gpu_tests.log 2>&1
tail -3 gpurun_out/r02a_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; tail -c 400 gpurun_out/r02a_bench.json
B='python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-time-to-tol'
$B > gpurun_out/r02a_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02a_launches_bicg.csv $B > /dev/null 2>&1
echo ncu rc=$?
