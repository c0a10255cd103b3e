# Round 2, call c: NAT kernels as compile-time variants (no spills); the concurrent-plans
# crash hunted with native backtraces; GPU suite; bench; ncu of C4 and C5.
set -x
mkdir -p gpurun_out
export GSK_SEGV_TRACE=1
for i in 1 2 3 4 5 6; do
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "concurrent" > gpurun_out/r02c_conc_$i.log 2>&1; echo "conc $i rc=$?"
done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02c_gpu_tests.log 2>&1; echo "suite rc=$?"
tail -3 gpurun_out/r02c_gpu_tests.log
timeout 600 python bench.py --no-time-to-tol > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; tail -c 300 gpurun_out/r02c_bench.json
python tools/prof_c4.py C4 > /dev/null && python tools/prof_c4.py C5 > /dev/null && \
ncu --set full --clock-control none --import-source on -k "regex:pass_kernel|gs_kernel" -c 40 -o /tmp/prof_c4 -f python tools/prof_c4.py C4 > gpurun_out/r02c_ncu_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:pass_kernel|gs_kernel" -c 40 -o /tmp/prof_c5 -f python tools/prof_c4.py C5 > gpurun_out/r02c_ncu_c5.log 2>&1
echo ncu rc=$?
python tools/ncu_detail.py /tmp/prof_c4.ncu-rep gpurun_out/r02_c4_v12_ncu_detail.json "ncu --set full, tools/prof_c4.py C4 sell (v12: natural-order SELL windows)" > gpurun_out/r02_c4_v12_ncu_detail.txt
python tools/ncu_detail.py /tmp/prof_c5.ncu-rep gpurun_out/r02_c5_v12_ncu_detail.json "ncu --set full, tools/prof_c4.py C5 sell (v12)" > gpurun_out/r02_c5_v12_ncu_detail.txt
python tools/ncu_traffic.py /tmp/prof_c4.ncu-rep gpurun_out/r02_ncu_traffic.json "ncu --set full --clock-control none, tools/prof_c4.py C4 sell, v12 engine (cold cache; per kernel the launch with the most DRAM bytes)" > /dev/null
