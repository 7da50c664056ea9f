#!/bin/bash
python gpurun_dbg.py 2>&1 | grep -v Warning | tail -8
timeout 300 python bench.py --config R4-small --steps 2 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R4small default', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['canonical_tflops_equiv'])"
timeout 600 python bench.py --config R4 --steps 1 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R4', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['canonical_tflops_equiv'])"
python bench.py --config R4-small --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_hex -s 0 -c 1 -o gpurun_out/hex_r4small_v6 python bench.py --config R4-small --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
