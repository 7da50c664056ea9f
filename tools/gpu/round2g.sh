mkdir -p gpurun_out/r2g; O=gpurun_out/r2g
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2>$O/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py > $O/bench_R4.json 2>$O/bench_R4.err; echo "R4 rc=$?"; cat $O/bench_R4.json
