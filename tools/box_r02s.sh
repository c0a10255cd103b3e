# Round 2, call s: persistent cooperative Bi-CGSTAB v2 (epoch flags, four-pass) — parity and timing.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "coop" > gpurun_out/r02s_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02s_tests.log
timeout 900 python tools/coop_timing.py gpurun_out/r02s_coop_timing.json > gpurun_out/r02s_coop_timing.log 2>&1; echo "timing rc=$?"
cat gpurun_out/r02s_coop_timing.log | tail -20
GSK_COOP_G=148 timeout 600 python tools/coop_timing.py gpurun_out/r02s_coop_timing_g148.json --cases=C2:256,C2:None,C3:64,C5:512 > gpurun_out/r02s_coop_timing_g148.log 2>&1
cat gpurun_out/r02s_coop_timing_g148.log | tail -8
