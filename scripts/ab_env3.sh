#!/bin/bash
# A/B/C of environment switches on the same box: ab_env3.sh reps "ENVA=1" "ENVB=1" ...
cd "$(dirname "$0")/.."
reps=$1; shift
for rep in $(seq 1 $reps); do
  for v in "" "$@"; do
    echo "[${v:-base}] $(env $v python bench.py --no-cpu-baseline --steps 50 ${BENCH_ARGS} 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), round(d["ms_per_step"],4), round(d["ms_per_step_device_span"],4), round(d["e2e"]["value"]/1e6,3))')"
  done
done
