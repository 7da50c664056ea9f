#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x 2>&1 | tail -4
python bench.py > gpurun_out/bench_r4.json 2> gpurun_out/bench_r4.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_r4.json
python bench.py --strategy blocked --no-cpu > gpurun_out/bench_r4_blocked.json 2> gpurun_out/bench_r4_blocked.err; echo "blocked rc=$?"; tail -c 800 gpurun_out/bench_r4_blocked.json; tail -3 gpurun_out/bench_r4_blocked.err
for c in R1 R3-16h; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2>/dev/null; echo "$c rc=$?"; done
