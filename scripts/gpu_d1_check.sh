mkdir -p gpurun_out
for K in 2 3 4; do
  timeout 600 python bench.py --config 4 --K $K --D 1 --steps 3 --warmup 3 --no-parity --exact-steps 0 --e2e-steps 0 > gpurun_out/d1_K$K.json 2> gpurun_out/d1_K$K.err
  python -c "import json; d=json.loads(open('gpurun_out/d1_K$K.json').read().strip().splitlines()[-1]); print('K=$K D=1', round(d['value'],3), round(d['ms_per_step'],1))"
done
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider -x -k "blob_config or overflow or shim or accumulate" > gpurun_out/pytest_sub.log 2>&1; tail -3 gpurun_out/pytest_sub.log
