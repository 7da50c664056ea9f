#!/bin/bash
# Delaunay (BASELINE #2) GPU checks + bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_delaunay.py -q -m gpu -rf -x > gpurun_out/pytest_delaunay.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_delaunay.log
timeout 600 python bench.py --config R2-small --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_R2-small.json 2> gpurun_out/bench_R2-small.err; echo "R2-small rc=$?"
timeout 900 python bench.py --config R2 --steps 3 --warmup 3 > gpurun_out/bench_R2.json 2> gpurun_out/bench_R2.err; echo "R2 rc=$?"
