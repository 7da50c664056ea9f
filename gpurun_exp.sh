#!/bin/bash
for v in default nofuse mb3; do
  if [ $v = default ]; then unset MF_LIB_PATH; else export MF_LIB_PATH=$PWD/paper_2101_08825_b200/_variants/$v/libmollifem_b200.so; fi
  timeout 300 python bench.py --config R4-small --steps 2 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['achieved'])"
done
unset MF_LIB_PATH
python -m pytest tests -q -m gpu -rf -k "hex" 2>&1 | tail -3
