# Round 2, call y: workspace cache — e2e breakdown, full GPU suite, default bench line.
set -x
mkdir -p gpurun_out
python tools/e2e_breakdown.py C4 > gpurun_out/r02y_e2e.log 2>&1; cat gpurun_out/r02y_e2e.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02y_tests.log 2>&1; echo "tests rc=$?"
tail -4 gpurun_out/r02y_tests.log
python bench.py > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r02y_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['frac'],d['roofline']['ms_per_launch'],d['e2e'],d['clocks'])"
