# Round 2, call w: what bounds the C5 SpMV passes — L1TEX / LTS throughput breakdowns and
# global-load requests vs sectors (ncu, C5 and C4 for contrast).
set -x
mkdir -p gpurun_out
python tools/prof_c4.py C5 > /dev/null 2>&1; echo "plain rc=$?"
M="gpu__time_duration.sum,dram__bytes.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,lts__t_sectors.sum,sm__cycles_elapsed.avg,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,breakdown:l1tex__throughput.avg.pct_of_peak_sustained_elapsed,breakdown:lts__throughput.avg.pct_of_peak_sustained_elapsed"
for C in C5 C4; do
ncu --clock-control none --metrics $M -k regex:pass_kernel -c 12 --csv python tools/prof_c4.py $C > gpurun_out/r02w_l1_$C.csv 2> gpurun_out/r02w_l1_$C.err; echo "ncu $C rc=$?"
done
wc -l gpurun_out/r02w_l1_*.csv
