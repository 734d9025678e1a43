# ncu captures of the render kernel: config 2 and config 3 at 512^2
mkdir -p gpurun_out
for C in 2 3; do
CMD="python bench.py --config $C --res 512 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/prof_plain_c$C.json 2> gpurun_out/prof_plain_c$C.err && \
ncu --set full --clock-control none --import-source on -k regex:k_render_rays -s 3 -c 1 -o gpurun_out/prof_render_c$C $CMD > gpurun_out/ncu_full_c$C.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_c$C.log
done
