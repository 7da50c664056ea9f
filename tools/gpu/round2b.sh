#!/bin/bash
# Round-2 (session 3) evidence: smoke, headline bench + reference arm, ncu
# launch list and full capture of the headline kernel, then the GPU suite.
mkdir -p gpurun_out/r2b
O=gpurun_out/r2b
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_R4.json 2> $O/bench_R4.err; echo "R4 rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_launches_R4.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hex2 --launch-skip 8 --launch-count 1 -f -o $O/hex2_R4small python bench.py --config R4-small --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_hex2.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:k_hex2 --launch-skip 8 --launch-count 1 -f -o $O/hex2_R4 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $O/ncu_hex2_R4.log 2>&1; echo "ncu full R4 rc=$?"
timeout 2400 python -m pytest tests -q -m gpu -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
