# work counters (ab/libkstats.so, -DSPHRAY_KSTATS=1) + plain timing + ncu full of the in-tree build
mkdir -p gpurun_out
for c in 2 3; do
  SPHRAY_B200_LIB=$PWD/ab/libkstats.so SPHRAY_TRACE=1 timeout 900 python bench.py --config $c --steps 1 --warmup 3 \
    --no-cpu-baseline --e2e-steps 0 > gpurun_out/kstats_c$c.json 2> gpurun_out/kstats_c$c.err
done
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
bash scripts/gpu_prof3.sh
