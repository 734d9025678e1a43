# parity suite + config-3 bench (3 steps) + config-2 trace
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
SPHRAY_TRACE=1 timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python - <<'PY'
import json
for c in (2, 3):
    try:
        d = json.loads(open(f"gpurun_out/bench_c{c}.json").read().strip().splitlines()[-1])
        print("c%d" % c, round(d["value"], 4), round(d["ms_per_step"], 1), "retries", d["stats"]["window_retries"])
    except Exception as e:
        print("c%d failed" % c, e)
PY
