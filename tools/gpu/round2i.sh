#!/bin/bash
# Final check of the round (session 4): smoke, the whole GPU suite, the
# driver's two bench arms, and fresh bench lines of the other workloads.
rm -f /tmp/ab_*.npy
mkdir -p gpurun_out/r2i; O=gpurun_out/r2i
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py > $O/bench_R4.json 2> $O/bench_R4.err; echo "R4 rc=$?"
for c in R2 R3-16h R1 R5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.json 2>$O/bench_$c.err; echo "$c rc=$?"; done
for c in $EXTRA_CFGS; do timeout 900 python bench.py --config $c --steps 1 --warmup 3 > $O/bench_$c.json 2>$O/bench_$c.err; echo "$c rc=$?"; done
