#!/bin/bash
# e2e of assemble() on R4 under several streaming layer splits / prefault
for pf in 0 1; do
for f in "" "0.6,0.9,1.0" "0.7,0.93,1.0"; do
  MF_PREFAULT=$pf MF_STREAM_FRACS=$f python tools/e2e_breakdown.py R4 2>&1 | tail -2 | sed "s/^/[pf=$pf $f] /"
done; done
