# config 4 order sweep: 4M blob, 1024^2, D in {1,2,3} x K in {1..4}
mkdir -p gpurun_out; rm -f gpurun_out/sweep_summary.txt
for D in 1 2 3; do for K in 1 2 3 4; do
  timeout 600 python bench.py --config 4 --K $K --D $D --steps 3 --warmup 3 --no-parity --exact-steps 0 --e2e-steps 0 \
    > gpurun_out/sweep_K${K}_D${D}.json 2> gpurun_out/sweep_K${K}_D${D}.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/sweep_K${K}_D${D}.json').read().strip().splitlines()[-1])
st=d['stats']; print('K=$K D=$D', round(d['value'],3), 'Mrays/s', round(d['ms_per_step'],1), 'ms', 'knots', st['knots'], 'knots/s %.3g' % (st['knots']/d['ms_per_step']*1e3), 'alu_frac %.3f' % d['alu_roofline']['frac'])" >> gpurun_out/sweep_summary.txt 2>&1 || echo "K=$K D=$D failed" >> gpurun_out/sweep_summary.txt
done; done
cat gpurun_out/sweep_summary.txt
