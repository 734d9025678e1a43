# A/B of library variants on one config (run under gpurun from repo root).
# VARIANTS="name|lib|bench args|ENV=v ...;..."  (lib "-" = in-tree build)
mkdir -p gpurun_out
CFG=${CFG:-3}
REPS=${REPS:-2}
VARIANTS=${VARIANTS:-"new|-|"}
for rep in $(seq 1 $REPS); do
  IFS=';' read -ra VS <<< "$VARIANTS"
  for v in "${VS[@]}"; do
    IFS='|' read -r name lib args envs <<< "$v"
    if [ "$lib" = "-" ]; then unset SPHRAY_B200_LIB; else export SPHRAY_B200_LIB=$PWD/$lib; fi
    timeout 900 env SPHRAY_TRACE=1 $envs python bench.py --config $CFG --steps 3 --warmup 3 --no-parity --exact-steps 0 --e2e-steps 0 $args \
      > gpurun_out/ab_${name}_${rep}.json 2> gpurun_out/ab_${name}_${rep}.err
    python - "$name" "$rep" <<'PY' >> gpurun_out/ab_summary.txt
import json,sys
try:
    d=json.loads(open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
    import re
    err = open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.err").read()
    shape = re.findall(r"cap=\d+ warps/cta=\d+ ctas/sm=\d+", err)
    print(sys.argv[1], sys.argv[2], round(d["value"],4), round(d["ms_per_step"],1), d.get("clocks",{}).get("sm_mhz"),
          "retries", d.get("stats",{}).get("window_retries"), shape[-1] if shape else "")
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
  done
done
cat gpurun_out/ab_summary.txt
