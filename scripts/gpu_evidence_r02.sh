# round-2 evidence pass (run under gpurun from the repo root):
#   default bench line, reference arm, launch list of one frame, ncu sections of
#   the render kernel at 2048^2 (hardware counters) and a full capture with
#   source at 512^2.
mkdir -p gpurun_out
cp paper_2401_02896_b200/build/render_d3.o gpurun_out/prof_render_d3.o
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench exit $?" >> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref exit $?" >> gpurun_out/bench_ref.err
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --exact-steps 0 --no-parity"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_default.csv $CMD > gpurun_out/ncu_launch.log 2>&1
SECTIONS="--section SpeedOfLight --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section Occupancy --section LaunchStats --section SchedulerStats --section WarpStateStats --section InstructionStats --metrics smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 1200 ncu $SECTIONS --clock-control none -k regex:k_render_rays -s 3 -c 1 \
  -o gpurun_out/render_2048 $CMD > gpurun_out/ncu_2048.log 2>&1
echo "ncu 2048 exit $?" >> gpurun_out/ncu_2048.log
CMD512="python bench.py --res 512 --steps 1 --warmup 3 --e2e-steps 0 --exact-steps 0 --no-parity"
$CMD512 > gpurun_out/prof_plain_512.json 2> gpurun_out/prof_plain_512.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_render_rays -s 3 -c 1 \
  -o gpurun_out/render_512 $CMD512 > gpurun_out/ncu_512.log 2>&1
echo "ncu 512 exit $?" >> gpurun_out/ncu_512.log
