mkdir -p gpurun_out
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --cpu-budget 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "c2 exit $?" >> gpurun_out/bench_c2.err
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --cpu-budget 10 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "c3 exit $?" >> gpurun_out/bench_c3.err
timeout 600 python bench.py --impl reference --config 2 --steps 2 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
echo "ref exit $?" >> gpurun_out/bench_ref_c2.err
