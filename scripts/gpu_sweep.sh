# occupancy sweep: register cap x knot window on config 3 at 1024^2
mkdir -p gpurun_out
: > gpurun_out/sweep.txt
for LIB in libsphray_b200.so libsphray_b200_r128.so; do
for WIN in 512 448 384 320 256; do
  SPHRAY_B200_LIB=$PWD/paper_2401_02896_b200/$LIB timeout 600 python bench.py --config 3 --res 1024 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --window $WIN > gpurun_out/sw.json 2>/dev/null
  python3 -c "
import json,sys
d=json.load(open('gpurun_out/sw.json'))
print('$LIB', $WIN, round(d['value'],4), round(d['breakdown_ms']['render_kernel'],1), d['stats']['window_retries'], d['stats']['max_window'])" >> gpurun_out/sweep.txt 2>&1
done; done
