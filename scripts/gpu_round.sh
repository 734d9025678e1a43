# full evidence pass: tests, default bench, reference arm, launch list, ncu capture
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench exit $?" >> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/launch_plain.json 2> gpurun_out/launch_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD3="python bench.py --config 3 --res 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD3 > gpurun_out/prof_plain_c3.json 2> gpurun_out/prof_plain_c3.err && \
ncu --set full --clock-control none --import-source on -k regex:k_render_rays -s 3 -c 1 -o gpurun_out/prof_render_c3 $CMD3 > gpurun_out/ncu_full_c3.log 2>&1
echo "done" >> gpurun_out/ncu_full_c3.log
