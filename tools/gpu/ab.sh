#!/bin/bash
# A/B: default library vs the variants named in $@ on one config ($CFG)
mkdir -p gpurun_out
CFG=${CFG:-R2}
for v in default "$@"; do
  if [ $v = default ]; then unset MF_LIB_PATH; else export MF_LIB_PATH=$PWD/paper_2101_08825_b200/_variants/$v/libmollifem_b200.so; fi
  timeout 600 python bench.py --config $CFG --steps ${STEPS:-2} --warmup 2 --no-cpu --no-e2e 2>gpurun_out/ab_$v.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $CFG', round(d['ms_per_step'],2), 'ms step', round(d['kernel_ms_per_step'],2), 'ms kernels', d['events'], round(d['roofline']['frac'],4))"
done
unset MF_LIB_PATH
