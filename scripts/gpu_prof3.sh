# ncu --set full capture (with source) of the render kernel on config 3 at 512^2;
# keeps the profiled object for the SASS -> source mapping (scripts/profile_report.py)
mkdir -p gpurun_out
cp paper_2401_02896_b200/build/render_d3.o gpurun_out/prof_render_d3.o
CMD="python bench.py --config 3 --res 512 --steps 1 --warmup 3 --no-parity --exact-steps 0 --e2e-steps 0"
$CMD > gpurun_out/prof_plain_c3.json 2> gpurun_out/prof_plain_c3.err && \
ncu --set full --clock-control none --import-source on -k regex:k_render_rays -s 3 -c 1 -o gpurun_out/prof_render_c3 $CMD > gpurun_out/ncu_full_c3.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_c3.log
