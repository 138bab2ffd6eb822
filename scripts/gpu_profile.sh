#!/bin/bash
# Round profile pass on the GPU box (run under gpurun, after the plain bench has
# exited 0): launch list of the bench, full-set capture of one c2 step, source
# page of the forward chain.  Everything lands in gpurun_out/ as CSV/JSON; the
# .ncu-rep files are dropped when they would blow gpurun's 64 MiB return limit.
# usage: scripts/gpu_profile.sh TAG      (e.g. r02g)
cd "$(dirname "$0")/.."
TAG=${1:-rXX}
O=gpurun_out
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${TAG}_c2_bench_launches_ncu.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
# one whole step (the second of three): skip the setup kernels by name
ncu --set full --clock-control none --import-source on \
    -k regex:"tc_fwd_chain|tc_bwd_chain|tc_gemm|k_zbias|k_qoi|k_sum_rows|k_refine|k_union|k_weights|k_seed|k_split|k_colsum|k_sel_colsum|k_finalize|k_export|k_step" \
    -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-70} -o $O/${TAG}_c2_step_full -f \
    python scripts/profile_step.py --steps 3 > $O/ncu_full.log 2>&1
python scripts/ncu_summary.py $O/${TAG}_c2_step_full.ncu-rep $O/${TAG}_c2_step_full_summary.json >> $O/ncu_full.log 2>&1
# source page (per-instruction samples and stall reasons) of the forward chain
ncu --set full --clock-control none --import-source on -k regex:"tc_fwd_chain" -s 1 -c 1 \
    -o $O/${TAG}_fwd_chain -f python scripts/profile_step.py --steps 3 > $O/ncu_src.log 2>&1
ncu -i $O/${TAG}_fwd_chain.ncu-rep --page source --csv > $O/${TAG}_fwd_chain_source.csv 2>> $O/ncu_src.log
ncu -i $O/${TAG}_fwd_chain.ncu-rep --page raw --csv > $O/${TAG}_fwd_chain_raw.csv 2>> $O/ncu_src.log
ncu --set full --clock-control none --import-source on -k regex:"tc_bwd_chain" -s 1 -c 1 \
    -o $O/${TAG}_bwd_chain -f python scripts/profile_step.py --steps 3 >> $O/ncu_src.log 2>&1
ncu -i $O/${TAG}_bwd_chain.ncu-rep --page source --csv > $O/${TAG}_bwd_chain_source.csv 2>> $O/ncu_src.log
for f in $O/*.ncu-rep; do
  [ -f "$f" ] && [ "$(stat -c %s "$f")" -gt 12000000 ] && rm -f "$f"
done
gzip -f $O/*_source.csv 2>/dev/null
du -sh $O
