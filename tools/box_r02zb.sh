# Round 2, call zb: what bounds the RCD passes at C4 — ncu --set full + L1TEX/LTS breakdowns.
set -x
mkdir -p gpurun_out
python tools/prof_c4.py C4 sell classes > /dev/null 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k "regex:pass_kernel" -c 24 -o /tmp/prof_rcd -f python tools/prof_c4.py C4 sell classes > gpurun_out/r02zb_ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_detail.py /tmp/prof_rcd.ncu-rep gpurun_out/r02zb_ncu_detail.json "ncu --set full, tools/prof_c4.py C4 sell classes (RCD NW=1)" > gpurun_out/r02zb_ncu_detail.txt
cat gpurun_out/r02zb_ncu_detail.txt
M="gpu__time_duration.sum,dram__bytes.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,lts__t_sectors.sum,sm__cycles_elapsed.avg,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,breakdown:l1tex__throughput.avg.pct_of_peak_sustained_elapsed,breakdown:lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_lsu.sum,sm__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"
ncu --clock-control none --metrics $M -k regex:pass_kernel -c 6 --csv python tools/prof_c4.py C4 sell classes > gpurun_out/r02zb_l1.csv 2> gpurun_out/r02zb_l1.err; echo "ncu rc=$?"
