#!/bin/bash
# Pack occupancy / priority sweep with the sparse bit volume.
python tools/dbg_opts.py pack_mode 0,1,2,3 c2 2>&1 | sed "s/^/bps=occ /"
for bps in 4 2; do
  SC_OPTS=pack_bps=$bps python tools/dbg_opts.py pack_mode 0,8,16,2,10,18 c2 2>&1 | sed "s/^/bps=$bps /"
done
