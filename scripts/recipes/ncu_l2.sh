# L2 op mix of the SSSP push kernels (reads vs RED vs ATOM sectors)
FAST="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra '' --no-ablation --no-configs --no-heavy"
M=gpu__time_duration.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_requests_op_red.sum,lts__t_requests_op_read.sum,lts__t_sectors.sum,lts__t_requests.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__d_sectors.sum,lts__t_sectors_srcunit_tex.sum,l1tex__m_xbar2l1tex_read_sectors.sum,smsp__inst_executed_op_global_red.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed
mkdir -p gpurun_out
for k in k_bm_large_pipe k_bm_twc k_bm_lb; do
eval timeout 900 ncu --metrics $M --clock-control none -k regex:$k -c 9 --csv --log-file gpurun_out/l2_$k.csv python bench.py $FAST > /dev/null 2>&1; echo "$k rc=$?"
done
