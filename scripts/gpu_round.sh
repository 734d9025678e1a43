# full evidence pass (run under gpurun from the repo root):
#   GPU parity suite, default bench line, reference arm, per-launch list,
#   DRAM traffic of the main render launch at the default workload, and an
#   ncu --set full capture of the render kernel (config 3 at 512^2).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench exit $?" >> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/launch_plain.json 2> gpurun_out/launch_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv $CMD > gpurun_out/ncu_launch.log 2>&1
SPHRAY_PROFILE_NO_RETRY=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:k_render_rays -s 3 -c 1 --csv --log-file gpurun_out/render_traffic.csv $CMD > gpurun_out/ncu_traffic.log 2>&1
bash scripts/gpu_prof3.sh
echo "done" >> gpurun_out/ncu_full_c3.log
