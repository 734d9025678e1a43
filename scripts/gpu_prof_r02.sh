# round-2 ncu evidence at the benchmarked workload (config 3, 2048^2), run under gpurun:
#   launch list of one frame (gpu__time_duration per kernel), DRAM bytes of the
#   render launch, and an ncu --set full capture (with source) of the render kernel.
mkdir -p gpurun_out
cp paper_2401_02896_b200/build/render_d3.o gpurun_out/prof_render_d3.o
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --exact-steps 0 --no-parity"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_default.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch.log
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_render_rays -s 3 -c 1 \
  -o gpurun_out/render_full_2048 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_full.log
ls -la gpurun_out/
