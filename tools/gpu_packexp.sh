#!/bin/bash
# Pack occupancy / loads-in-flight sweep (pack_bps x pack_mode U bits).
for bps in 0 4 2 1; do
  SC_OPTS=pack_bps=$bps python tools/dbg_opts.py pack_mode 0,8,16 c2 c5 2>&1 | sed "s/^/bps=$bps /"
done
