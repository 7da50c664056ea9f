#!/bin/bash
# e2e of assemble() on R4 under several streaming layer splits
for f in "" "0.5,0.8,0.95,1.0" "0.6,0.9,1.0" "0.35,0.65,0.85,0.96,1.0"; do
  MF_STREAM_FRACS=$f python tools/e2e_breakdown.py R4 2>&1 | tail -2 | sed "s/^/[$f] /"
done
