# hardware counters of the render kernel at the benchmarked 2048^2 workload
# (explicit metric list: no instrumented passes, which do not finish on a 4 s launch)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --exact-steps 0 --no-parity"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__inst_executed.avg.per_cycle_active,sm__instruction_throughput.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,launch__registers_per_thread,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg"
$CMD > gpurun_out/m2048_plain.json 2> gpurun_out/m2048_plain.err
timeout 900 ncu --metrics $M --clock-control none -k regex:k_render_rays -s 3 -c 1 -o gpurun_out/render_2048_metrics $CMD > gpurun_out/ncu_m2048.log 2>&1
echo "ncu metrics exit $?" >> gpurun_out/ncu_m2048.log
