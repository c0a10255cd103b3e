# Round 2, call zf: RCD stencil slots (+-1 by shuffle, +-256 from the neighbouring windows) — parity, bench, L1 wavefronts.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "row_classes or class_slots" > gpurun_out/r02zf_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02zf_tests.log
for v in slots noslots; do
  if [ $v = slots ]; then unset GSK_RCD_SLOTS; else export GSK_RCD_SLOTS=0; fi
  for cfg in C4 C3; do
    python bench.py --config $cfg --no-e2e --no-cpu --no-time-to-tol --no-plain-compare > gpurun_out/r02zf_${cfg}_$v.json 2> gpurun_out/r02zf_${cfg}_$v.err
  done
done
unset GSK_RCD_SLOTS
for f in gpurun_out/r02zf_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); x = d["extra"]
    print(sys.argv[1], round(d["value"], 1), "bicg", round(x["bicgstab"]["iters_per_s"], 1), x["bicgstab"]["iterations"], "gmres", round(x["gmres"]["iters_per_s"], 1), "spmv", round(x["spmv"]["ms"], 4), {k: round(v, 4) for k, v in x["probe_ms"].items() if v}, d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
M="gpu__time_duration.sum,dram__bytes.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors.sum,sm__cycles_elapsed.avg,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_lsu.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"
ncu --clock-control none --metrics $M -k regex:pass_kernel -c 6 --csv python tools/prof_c4.py C4 sell classes > gpurun_out/r02zf_l1.csv 2> gpurun_out/r02zf_l1.err; echo "ncu rc=$?"
