#!/bin/bash
# k_tet A/B: lean state (scatter geometry / G out of registers), 3 blocks/SM,
# outer-point unroll, batched leaf classification
rm -f /tmp/ab_*.npy; df -h /tmp | tail -1
mkdir -p gpurun_out/r2h; O=gpurun_out/r2h
V=paper_2101_08825_b200/_variants
L="paper_2101_08825_b200/_lib/libmollifem_b200.so"
for v in "$@"; do L="$L $V/$v/libmollifem_b200.so"; done
timeout 1500 python tools/ab_time.py --config R4-tet --reps 1 $L 2>&1 | cut -c1-220 | tee $O/ab_R4tet.log
timeout 900 python tools/ab_time.py --config R5-tet-small --reps 2 $L 2>&1 | cut -c1-220 | tee $O/ab_R5tetsmall.log
# parity of the candidate default (first variant that is to ship) on the tet tests
if [ -n "$CHECK" ]; then
  MF_LIB_PATH=$PWD/$V/$CHECK/libmollifem_b200.so timeout 1200 python -m pytest tests/test_tet.py tests/test_tet_composite.py tests/test_gpu_baseline_parity.py -m gpu -x -q -k "tet" > $O/pytest_tet_$CHECK.txt 2>&1; echo "pytest $CHECK rc=$?"; tail -3 $O/pytest_tet_$CHECK.txt
fi
