#!/bin/bash
# Round evidence on the GPU box: bench lines (with clocks) for the BASELINE
# workloads, the reference arm, the ncu launch list of one R4 step and one
# ncu --set full capture of the dominant kernel.  Usage:
#   tools/evidence.sh OUTDIR [configs...]
OUT=${1:-gpurun_out/ev}; shift
mkdir -p $OUT
CFGS=${@:-"R4 R2 R3-16h R4-tet R5-tet-64 R1 R1-tri3 R4-gauss2"}
for c in $CFGS; do
  extra=""
  case $c in R4) extra="--steps 5 --warmup 3";; R4-tet|R5-tet-64) extra="--steps 2 --warmup 3 --e2e-steps 1";; *) extra="--steps 5 --warmup 3";; esac
  timeout 1200 python bench.py --config $c $extra > $OUT/bench_$c.log 2>&1
  tail -1 $OUT/bench_$c.log > $OUT/bench_$c.json
done
timeout 900 python bench.py --config R4 --strategy blocked --steps 5 --warmup 3 --no-cpu > $OUT/bench_R4_blocked.log 2>&1; tail -1 $OUT/bench_R4_blocked.log > $OUT/bench_R4_blocked.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref.log 2>&1; tail -1 $OUT/bench_ref.log > $OUT/bench_ref.json
