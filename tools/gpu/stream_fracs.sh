#!/bin/bash
# e2e of assemble() on R4 under several streaming layer splits
for f in "" "0.9,1.0" "0.8,0.95,1.0" "0.93,1.0"; do
  MF_STREAM_FRACS=$f python tools/e2e_breakdown.py R4 2>&1 | grep "trial [12]" | sed "s/^/[$f] /"
done
