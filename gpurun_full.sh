#!/bin/bash
# full round check: tests, bench (ours + reference arm), launch list, ncu
mkdir -p gpurun_out
python -m pytest tests -q -m gpu 2>&1 | tail -4
python bench.py > gpurun_out/bench_r4.json 2> gpurun_out/bench_r4.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_r4.json
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
for c in R1 R3-16h; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2>/dev/null; echo "$c rc=$?"; done
python bench.py --config R4-small --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r4small.csv python bench.py --config R4-small --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_hex -s 0 -c 1 -o gpurun_out/hex_r4small_v5 python bench.py --config R4-small --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
