# Round 2, final measurement of the v18 engine (row-class dictionary + stencil slots as the
# default SELL plan encoding): bench line, launch lists of the bench command, ncu --set full
# of C4, per-config table, full-size and paper parity on the default encoding, GPU suite.
set -x
TAG=r02_c4_v18
mkdir -p gpurun_out
python bench.py > gpurun_out/r02_bench_v18.json 2> gpurun_out/r02_bench_v18.err; echo "bench rc=$?"
B='python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-time-to-tol --no-plain-compare'
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches_bicg.csv $B > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 13000 -c 800 --csv --log-file gpurun_out/${TAG}_launches_gmres.csv $B > /dev/null 2>&1
echo "launch lists rc=$?"
python tools/launch_share.py gpurun_out/${TAG}_launches_bicg.csv gpurun_out/${TAG}_launches_gmres.csv > gpurun_out/${TAG}_launches_share.txt
python tools/prof_c4.py C4 sell classes > /dev/null && \
ncu --set full --clock-control none --import-source on -k "regex:pass_kernel|gs_kernel" -c 40 -o /tmp/prof_c4 -f python tools/prof_c4.py C4 sell classes > gpurun_out/${TAG}_ncu_c4.log 2>&1
echo "ncu rc=$?"
python tools/ncu_detail.py /tmp/prof_c4.ncu-rep gpurun_out/${TAG}_ncu_detail.json "ncu --set full, tools/prof_c4.py C4 sell classes ($TAG)" > gpurun_out/${TAG}_ncu_detail.txt
python tools/ncu_traffic.py /tmp/prof_c4.ncu-rep gpurun_out/r02_ncu_traffic_rcd.json "ncu --set full --clock-control none, tools/prof_c4.py C4 sell classes, $TAG (cold cache; per kernel the launch with the most DRAM bytes)" > /dev/null
cat gpurun_out/${TAG}_ncu_detail.txt
timeout 1500 python tools/run_configs.py gpurun_out/r02_configs_v18 C1 C3 C4 > gpurun_out/${TAG}_configs.log 2>&1; echo "configs rc=$?"
timeout 2400 python tools/full_parity.py gpurun_out/r02_full_parity.json > gpurun_out/${TAG}_full_parity.log 2>&1; echo "full parity rc=$?"
timeout 1200 python tools/full_parity.py --paper gpurun_out/r02_paper_parity.json > gpurun_out/${TAG}_paper_parity.log 2>&1; echo "paper parity rc=$?"
timeout 3000 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/${TAG}_tests.log
python -c "
import __graft_entry__ as g; g.smoke()"
ls gpurun_out | grep -E "v18|parity|rcd"
