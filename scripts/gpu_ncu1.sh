mkdir -p gpurun_out
CMD="python bench.py --config 2 --res 256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_256.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_render_rays -s 3 -c 1 -o gpurun_out/prof_render_c2_256 $CMD > gpurun_out/ncu_full.log 2>&1
echo done >> gpurun_out/ncu_full.log
