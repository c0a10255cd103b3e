# Round 2, call z: row-class dictionary (RCD) — parity tests, then C4 / C3 bench lines plain vs classes.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "row_classes" > gpurun_out/r02z_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02z_tests.log
for si in classes plain; do
python bench.py --no-e2e --no-cpu --no-time-to-tol --sell-index $si > gpurun_out/r02z_bench_$si.json 2> gpurun_out/r02z_bench_$si.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r02z_bench_$si.json').read().strip().splitlines()[-1]);print('$si', d['value'],d['roofline']['ms_per_launch'],d['extra']['probe_ms'],d['extra']['spmv']['ms'],d['extra']['bicgstab']['iters_per_s'],d['extra']['gmres']['iters_per_s'],d['extra']['steps_ms'][-1])"
python bench.py --config C3 --no-e2e --no-cpu --no-time-to-tol --sell-index $si > gpurun_out/r02z_bench_c3_$si.json 2> gpurun_out/r02z_bench_c3_$si.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r02z_bench_c3_$si.json').read().strip().splitlines()[-1]);print('C3 $si', d['value'],d['extra']['probe_ms'],d['extra']['spmv']['ms'],d['extra']['bicgstab']['iters_per_s'],d['extra']['gmres']['iters_per_s'])"
done
