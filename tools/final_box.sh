set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
python bench.py > gpurun_out/r01_bench_default.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/r01_bench_default.json
B='python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-time-to-tol'
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01_c4_v11_launches_bicg.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 13000 -c 800 --csv --log-file gpurun_out/r01_c4_v11_launches_gmres.csv $B > /dev/null 2>&1
bash tools/ncu_box_c4.sh > /dev/null 2>&1; echo ncu rc=$?
