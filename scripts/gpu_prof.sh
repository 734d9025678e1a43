# parity suite + ncu capture of the render kernel (config 2 at 512^2)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
CMD="python bench.py --config 2 --res 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:k_render_rays -s 3 -c 1 -o gpurun_out/prof_render $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full.log
