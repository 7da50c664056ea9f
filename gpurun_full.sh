#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -rf 2>&1 | tail -6 > gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_r4.json 2> gpurun_out/bench_r4.err; echo "bench rc=$?"
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo "ref rc=$?"
python bench.py --strategy blocked --no-cpu > gpurun_out/bench_r4_blocked.json 2> /dev/null; echo "blocked rc=$?"
for c in R1 R3-2h R3-4h R3-8h R3-16h R4-gauss2; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2>/dev/null; echo "$c rc=$?"; done
python bench.py --config R4 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_hex -c 8 --csv --log-file gpurun_out/launches_r4_hex.csv python bench.py --config R4 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
