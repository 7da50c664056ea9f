mkdir -p gpurun_out/r2e; O=gpurun_out/r2e
V=paper_2101_08825_b200/_variants; L=paper_2101_08825_b200/_lib/libmollifem_b200.so
timeout 600 python tools/ab_time.py --config R2 --reps 2 $L $V/triq_b2/libmollifem_b200.so $V/triq_b3/libmollifem_b200.so $V/triq_scan/libmollifem_b200.so 2>&1 | cut -c1-150 | tee $O/ab26.log
timeout 2400 python -m pytest tests -q -m gpu -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_R4.json 2> $O/bench_R4.err; echo "R4 rc=$?"
timeout 600 python bench.py --strategy blocked --no-cpu > $O/bench_R4_blocked.json 2>/dev/null; echo "blocked rc=$?"
