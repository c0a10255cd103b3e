# Round 2, call r: re-validation of HEAD after the container re-creation — full GPU suite,
# smoke and the default bench line.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02r_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/r02r_tests.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/r02r_tests.log
python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r02r_bench.json
