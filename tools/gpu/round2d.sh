#!/bin/bash
# Final check of the round: smoke, the GPU suite, the driver's two bench
# arms, and the full-size BASELINE #5 workloads for the record.
mkdir -p gpurun_out/r2d
O=gpurun_out/r2d
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py > $O/bench_R4.json 2> $O/bench_R4.err; echo "R4 rc=$?"
timeout 900 python bench.py --config R5 --steps 2 --warmup 3 --no-cpu > $O/bench_R5.json 2> $O/bench_R5.err; echo "R5 rc=$?"
timeout 1500 python bench.py --config R5-tet --steps 1 --warmup 3 --no-cpu > $O/bench_R5-tet.json 2> $O/bench_R5-tet.err; echo "R5-tet rc=$?"
