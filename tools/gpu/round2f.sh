#!/bin/bash
# tet bench lines after the 2-blocks/SM change + ncu summary of the shipped k_tet
rm -f /tmp/ab_*.npy
mkdir -p gpurun_out/r2f; O=gpurun_out/r2f
timeout 900 python -m pytest tests/test_tet.py tests/test_tet_composite.py tests/test_gpu_baseline_parity.py -m gpu -x -q -k tet > $O/pytest_tet.txt 2>&1; echo "pytest tet rc=$?"; tail -2 $O/pytest_tet.txt
for c in R4-tet R5-tet-64; do timeout 900 python bench.py --config $c --steps 1 --warmup 3 > $O/bench_$c.json 2>$O/bench_$c.err; echo "$c rc=$?"; done
timeout 1500 python bench.py --config R5-tet --steps 1 --warmup 3 --no-cpu > $O/bench_R5-tet.json 2> $O/bench_R5-tet.err; echo "R5-tet rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:^k_tet$" --launch-skip 100 --launch-count 1 -f -o $O/ktet_R4tet python bench.py --config R4-tet --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_ktet.log 2>&1; echo "ncu tet rc=$?"
