#!/bin/bash
# k_tet: explicit shared-memory carve-out A/B on R4-tet
rm -f /tmp/ab_*.npy
mkdir -p gpurun_out/r2j; O=gpurun_out/r2j
timeout 900 python tools/ab_time.py --config R4-tet --reps 1 paper_2101_08825_b200/_lib/libmollifem_b200.so paper_2101_08825_b200/_variants/tet_carve/libmollifem_b200.so 2>&1 | cut -c1-200 | tee $O/ab_carve_R4tet.log
timeout 600 python tools/ab_time.py --config R5-tet-small --reps 2 paper_2101_08825_b200/_lib/libmollifem_b200.so paper_2101_08825_b200/_variants/tet_carve/libmollifem_b200.so 2>&1 | cut -c1-200 | tee $O/ab_carve_R5tetsmall.log
