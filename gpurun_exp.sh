#!/bin/bash
# exploratory timings (not bench values)
for v in default mb4 b1 mb2; do
  if [ $v = default ]; then unset MF_LIB_PATH; else export MF_LIB_PATH=$PWD/paper_2101_08825_b200/_variants/$v/libmollifem_b200.so; fi
  timeout 300 python bench.py --config R4-small --steps 2 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['canonical_tflops_equiv'])"
done
unset MF_LIB_PATH
for c in R1 R3-16h R3-2h; do timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['canonical_tflops_equiv'])"; done
python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --config R4 --steps 1 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R4', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['canonical_tflops_equiv'])"
python bench.py --config R4-small --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_hex -s 0 -c 1 -o gpurun_out/hex_r4small_v4 python bench.py --config R4-small --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu.log 2>&1
tail -1 gpurun_out/ncu.log
