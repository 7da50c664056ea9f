#!/bin/bash
# last sanity of the final library: smoke + the tet parity tests + one R4-tet-small bench line
mkdir -p gpurun_out/r2k; O=gpurun_out/r2k
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python -m pytest tests/test_tet.py tests/test_tet_composite.py tests/test_gpu_baseline_parity.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_subset.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_subset.txt
