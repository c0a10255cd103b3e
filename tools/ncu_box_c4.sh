# On the GPU box: ncu --set full of tools/prof_c4.py (C4, top kernels), summarised on
# the box (the raw report is too large to bring back).  TAG names the round/version.
set -e
TAG=${TAG:-r01_c4_v11}
mkdir -p gpurun_out
python tools/prof_c4.py > /dev/null
ncu --set full --clock-control none -k "regex:pass_kernel|mdot_pass|gs_kernel" -c 60 -o /tmp/prof_$TAG -f python tools/prof_c4.py > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_$TAG.ncu-rep > gpurun_out/${TAG}_ncu_full.txt
python tools/ncu_traffic.py /tmp/prof_$TAG.ncu-rep gpurun_out/r01_ncu_traffic.json "ncu --set full --clock-control none, tools/prof_c4.py (C4 256^3, GS(2), SELL-C-32-256), report prof_$TAG (cold cache; per kernel the launch with the most DRAM bytes)" > gpurun_out/traffic.log
ls -la gpurun_out
