# work counters: build with `scripts/build_variants.sh kstats "-DSPHRAY_KSTATS=1"`,
# then run under gpurun from the repo root (SPHRAY_TRACE=1 prints the counters)
mkdir -p gpurun_out
for c in 2 3; do
  SPHRAY_B200_LIB=$PWD/build_variants/libkstats.so SPHRAY_TRACE=1 timeout 900 python bench.py --config $c \
    --steps 1 --warmup 3 --no-parity --exact-steps 0 --e2e-steps 0 > gpurun_out/kstats_c$c.json 2> gpurun_out/kstats_c$c.err
done
