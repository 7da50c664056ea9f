#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -rf 2>&1 | tail -6 > gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_r4.json 2> gpurun_out/bench_r4.err; echo "bench rc=$?"
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo "ref rc=$?"
python bench.py --strategy blocked --no-cpu > gpurun_out/bench_r4_blocked.json 2> /dev/null; echo "blocked rc=$?"
for c in R1 R3-2h R3-16h; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2>/dev/null; echo "$c rc=$?"; python bench.py --config $c --strategy blocked --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_${c}_blocked.json 2>/dev/null; done
