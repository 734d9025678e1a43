# compute-sanitizer memcheck / racecheck over a few small GPU parity tests
# (every kernel variant: production, robust, dumps, retry, degree 1, large TF)
mkdir -p gpurun_out
K="render_matches_reference or small_window_retry or degree_one or large_transfer or field_pieces or sharded"
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "$K" > gpurun_out/sanitize_memcheck.log 2>&1
echo "memcheck exit $?" >> gpurun_out/sanitize_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "render_matches_reference and desk" > gpurun_out/sanitize_racecheck.log 2>&1
echo "racecheck exit $?" >> gpurun_out/sanitize_racecheck.log
