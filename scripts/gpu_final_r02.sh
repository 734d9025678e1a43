# round-2 final evidence, part A (run under gpurun from the repo root):
# default bench line, reference arm, config-1/2 lines, launch list of one
# frame, hardware counters of the render kernel at 2048^2.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench exit $?" >> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref exit $?" >> gpurun_out/bench_ref.err
for c in 1 2; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "config $c exit $?" >> gpurun_out/bench_c$c.err
done
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --exact-steps 0 --no-parity"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_default.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/ncu_launch.log
bash scripts/gpu_metrics_2048.sh
