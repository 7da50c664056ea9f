#!/bin/bash
# k_tet: whole-library A/B of the variants named in $@ on R4-tet / R5-tet-small
rm -f /tmp/ab_*.npy
mkdir -p gpurun_out/r2j; O=gpurun_out/r2j
L="paper_2101_08825_b200/_lib/libmollifem_b200.so"
for v in "$@"; do L="$L paper_2101_08825_b200/_variants/$v/libmollifem_b200.so"; done
timeout 900 python tools/ab_time.py --config R4-tet --reps 1 $L 2>&1 | cut -c1-200 | tee $O/ab_R4tet.log
timeout 600 python tools/ab_time.py --config R5-tet-small --reps 2 $L 2>&1 | cut -c1-200 | tee $O/ab_R5tetsmall.log
