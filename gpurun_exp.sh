#!/bin/bash
for v in default mb3 mb2; do
  if [ $v = default ]; then unset MF_LIB_PATH; else export MF_LIB_PATH=$PWD/paper_2101_08825_b200/_variants/$v/libmollifem_b200.so; fi
  for c in R3-16h R1; do
  timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', d['ms_per_step'], d['roofline']['achieved'])"
  done
done
unset MF_LIB_PATH
python -m pytest tests -q -m gpu -rf -k "tri or quad or R1" 2>&1 | tail -3
