#!/bin/bash
for v in default old2d; do
  if [ $v = default ]; then unset MF_LIB_PATH; else export MF_LIB_PATH=$PWD/paper_2101_08825_b200/_variants/$v/libmollifem_b200.so; fi
  for c in R1 R3-2h R3-16h; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', d['ms_per_step'])"
  done
done
unset MF_LIB_PATH
timeout 300 python bench.py --config R4-small --steps 2 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R4-small prefetch', d['ms_per_step'])"
timeout 600 python bench.py --config R4 --steps 1 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R4 prefetch', d['ms_per_step'])"
python -m pytest tests/test_gpu_parallel.py -q -rf 2>&1 | tail -3
