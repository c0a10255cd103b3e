# Round 2: measurement of the current engine (v13) — launch list of the bench command,
# ncu --set full of C4 / C5, emulated sharding, the paper tables.  TAG names it.
set -x
TAG=${TAG:-r02_c4_v13}
mkdir -p gpurun_out
B='python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-time-to-tol'
for P in 2 8; do python bench.py --shards $P --steps 2 --warmup 3 --no-e2e > gpurun_out/${TAG}_shards$P.json 2>&1; done
timeout 900 python tools/paper_tables.py gpurun_out/r02_paper_tables > gpurun_out/${TAG}_paper_tables.log 2>&1; echo "paper rc=$?"
$B > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches_bicg.csv $B > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 13000 -c 800 --csv --log-file gpurun_out/${TAG}_launches_gmres.csv $B > /dev/null 2>&1 && \
python tools/prof_c4.py C4 > /dev/null && python tools/prof_c4.py C5 > /dev/null && \
ncu --set full --clock-control none --import-source on -k "regex:pass_kernel|gs_kernel" -c 40 -o /tmp/prof_c4 -f python tools/prof_c4.py C4 > gpurun_out/${TAG}_ncu_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:pass_kernel|gs_kernel" -c 40 -o /tmp/prof_c5 -f python tools/prof_c4.py C5 > gpurun_out/${TAG}_ncu_c5.log 2>&1
echo "ncu rc=$?"
python tools/launch_share.py gpurun_out/${TAG}_launches_bicg.csv gpurun_out/${TAG}_launches_gmres.csv > gpurun_out/${TAG}_launches_share.txt
python tools/ncu_detail.py /tmp/prof_c4.ncu-rep gpurun_out/${TAG}_ncu_detail.json "ncu --set full, tools/prof_c4.py C4 sell ($TAG)" > gpurun_out/${TAG}_ncu_detail.txt
python tools/ncu_detail.py /tmp/prof_c5.ncu-rep gpurun_out/r02_c5_v13_ncu_detail.json "ncu --set full, tools/prof_c4.py C5 sell ($TAG)" > gpurun_out/r02_c5_v13_ncu_detail.txt
python tools/ncu_traffic.py /tmp/prof_c4.ncu-rep gpurun_out/r02_ncu_traffic.json "ncu --set full --clock-control none, tools/prof_c4.py C4 sell, $TAG (cold cache; per kernel the launch with the most DRAM bytes)" > /dev/null
ls gpurun_out | grep $TAG
