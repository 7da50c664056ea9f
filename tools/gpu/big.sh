#!/bin/bash
mkdir -p gpurun_out/final
timeout 900 python bench.py > gpurun_out/final/bench_r4.json 2> gpurun_out/final/bench_r4.err; echo "R4 rc=$?"
timeout 600 python bench.py --config R2 --steps 3 --warmup 3 > gpurun_out/final/bench_R2.json 2>/dev/null; echo "R2 rc=$?"
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/final/mem.txt
free -g >> gpurun_out/final/mem.txt
timeout 1800 python bench.py --config R5-tet --steps 1 --warmup 3 --no-e2e > gpurun_out/final/bench_R5-tet.json 2> gpurun_out/final/bench_R5-tet.err; echo "R5-tet rc=$?"
