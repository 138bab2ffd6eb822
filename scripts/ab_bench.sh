#!/bin/bash
# A/B of two builds of the library on the same box: ab_bench.sh VARIANT...
# (each paper_2305_20053_b200/libsaadino_<VARIANT>.so is swapped in turn)
cd "$(dirname "$0")/.."
cp paper_2305_20053_b200/libsaadino.so /tmp/libsaadino.orig.so
for rep in 1 2; do
  for v in "$@"; do
    cp "paper_2305_20053_b200/libsaadino_$v.so" paper_2305_20053_b200/libsaadino.so
    echo "$v $(python bench.py --no-cpu-baseline --steps 50 ${BENCH_ARGS} 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), round(d["ms_per_step"],4), round(d["e2e"]["value"]/1e6,3))')"
  done
done
cp /tmp/libsaadino.orig.so paper_2305_20053_b200/libsaadino.so
