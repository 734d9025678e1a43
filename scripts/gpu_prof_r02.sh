# round-2 ncu evidence at the benchmarked workload (config 3), run under gpurun:
#   (1) hardware-counter sections of the render kernel at 2048^2 (no source
#       counters: instrumented SASS passes do not finish on a 4 s launch),
#   (2) a full capture with source counters at 512^2 (same kernel, same scene).
mkdir -p gpurun_out
cp paper_2401_02896_b200/build/render_d3.o gpurun_out/prof_render_d3.o
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --exact-steps 0 --no-parity"
SECTIONS="--section SpeedOfLight --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section Occupancy --section LaunchStats --section SchedulerStats --section WarpStateStats --section InstructionStats --metrics smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__pcsamp_warps_issue_stalled_wait"
timeout 1200 ncu $SECTIONS --clock-control none -k regex:k_render_rays -s 3 -c 1 \
  -o gpurun_out/render_2048 $CMD > gpurun_out/ncu_2048.log 2>&1
echo "ncu 2048 exit $?" >> gpurun_out/ncu_2048.log
CMD512="python bench.py --res 512 --steps 1 --warmup 3 --e2e-steps 0 --exact-steps 0 --no-parity"
$CMD512 > gpurun_out/prof_plain_512.json 2> gpurun_out/prof_plain_512.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_render_rays -s 3 -c 1 \
  -o gpurun_out/render_512 $CMD512 > gpurun_out/ncu_512.log 2>&1
echo "ncu 512 exit $?" >> gpurun_out/ncu_512.log
