#!/bin/bash
# A/B of an environment switch on the same box: ab_env.sh "ENV=1" [reps]
cd "$(dirname "$0")/.."
for rep in $(seq 1 ${2:-3}); do
  for v in "" "$1"; do
    echo "[${v:-base}] $(env $v python bench.py --no-cpu-baseline --steps 50 ${BENCH_ARGS} 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), round(d["ms_per_step"],4), round(d["ms_per_step_device_span"],4), round(d["e2e"]["value"]/1e6,3))')"
  done
done
