#!/bin/bash
mkdir -p gpurun_out/final
timeout 1800 python -m pytest tests -q -m gpu -rf > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/final/bench_r4.json 2> gpurun_out/final/bench_r4.err; echo "R4 rc=$?"
timeout 600 python bench.py --config R2 --steps 3 --warmup 3 > gpurun_out/final/bench_R2.json 2>/dev/null; echo "R2 rc=$?"
timeout 600 python bench.py --config R3-16h --steps 3 --warmup 3 > gpurun_out/final/bench_R3-16h.json 2>/dev/null; echo "R3-16h rc=$?"
