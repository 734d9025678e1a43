# round-2 final evidence, part B: the GPU test suite, then a --set full
# capture (with source) of the render kernel at 512^2 for the stall reasons.
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
cp paper_2401_02896_b200/build/render_d3.o gpurun_out/prof_render_d3.o
CMD512="python bench.py --res 512 --steps 1 --warmup 3 --e2e-steps 0 --exact-steps 0 --no-parity"
$CMD512 > gpurun_out/prof_plain_512.json 2> gpurun_out/prof_plain_512.err
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_render_rays -s 3 -c 1 \
  -o gpurun_out/render_512 $CMD512 > gpurun_out/ncu_512.log 2>&1
echo "ncu 512 exit $?" >> gpurun_out/ncu_512.log
