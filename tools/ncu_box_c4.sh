set -e
mkdir -p gpurun_out
python tools/prof_c4.py > /dev/null
ncu --set full --clock-control none -k "regex:pass_kernel|mdot_pass|gs_kernel" -c 60 -o /tmp/prof_c4_v8 -f python tools/prof_c4.py > gpurun_out/ncu_c4_v6.log 2>&1
python tools/ncu_summary.py /tmp/prof_c4_v8.ncu-rep > gpurun_out/r01_c4_v8_ncu_full.txt
python tools/ncu_traffic.py /tmp/prof_c4_v8.ncu-rep gpurun_out/r01_ncu_traffic.json "ncu --set full --clock-control none, tools/prof_c4.py (C4 256^3, GS(2), SELL-C-32-256), report prof_c4_v8 (cold cache; per kernel the launch with the most DRAM bytes)" > gpurun_out/traffic.log
ls -la gpurun_out
