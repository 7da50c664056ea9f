python tools/step_breakdown.py R2-small 2>&1 | tail -2
nvidia-smi --query-gpu=index,clocks.sm --format=csv,noheader -lms 200 > /dev/null 2>&1 &
NP=$!
python tools/step_breakdown.py R2-small 2>&1 | tail -2
kill $NP
CFG=R2-small STEPS=3 bash tools/gpu/ab.sh pool
