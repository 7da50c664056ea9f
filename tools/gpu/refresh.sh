#!/bin/bash
# Round evidence: GPU tests, smoke, headline bench (+ reference arm), every
# workload's bench line.
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -q -m gpu -rf > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/final/bench_r4.json 2> gpurun_out/final/bench_r4.err; echo "R4 rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --strategy blocked --no-cpu > gpurun_out/final/bench_r4_blocked.json 2>/dev/null; echo "blocked rc=$?"
for c in R1 R1-tri3 R2 R2-small R3-2h R3-16h; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/final/bench_$c.json 2>/dev/null; echo "$c rc=$?"; done
for c in R1 R3-2h R3-16h; do timeout 600 python bench.py --config $c --strategy blocked --steps 3 --warmup 3 --no-cpu > gpurun_out/final/bench_${c}_blocked.json 2>/dev/null; echo "$c blocked rc=$?"; done
for c in R4-tet R5-tet-64; do timeout 900 python bench.py --config $c --steps 1 --warmup 3 --no-e2e > gpurun_out/final/bench_$c.json 2>/dev/null; echo "$c rc=$?"; done
