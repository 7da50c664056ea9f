#!/bin/bash
# Round-2 (session 3) evidence for the other workloads: bench lines with
# clocks, and fresh ncu --set full captures of the shipped k_tri_q / k_tet /
# k_2d builds.
mkdir -p gpurun_out/r2c
O=gpurun_out/r2c
for c in R1 R1-tri3 R2 R2-small R3-2h R3-16h R4-gauss2 R4-small; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2>$O/bench_$c.err; echo "$c rc=$?"; done
timeout 600 python bench.py --strategy blocked --no-cpu > $O/bench_R4_blocked.json 2>/dev/null; echo "blocked rc=$?"
for c in R4-tet R5-tet-64; do timeout 900 python bench.py --config $c --steps 1 --warmup 3 > $O/bench_$c.json 2>$O/bench_$c.err; echo "$c rc=$?"; done
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:^k_tri_q$" --launch-skip 40 --launch-count 1 -f -o $O/ktriq_R2 python bench.py --config R2 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_ktriq.log 2>&1; echo "ncu triq rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:^k_tet$" --launch-skip 100 --launch-count 1 -f -o $O/ktet_R4tet python bench.py --config R4-tet --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_ktet.log 2>&1; echo "ncu tet rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:^k_2d$" --launch-skip 6 --launch-count 1 -f -o $O/k2d_R3 python bench.py --config R3-16h --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_k2d.log 2>&1; echo "ncu 2d rc=$?"
