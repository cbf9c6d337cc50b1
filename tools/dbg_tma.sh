#!/bin/bash
# TMA pack: correctness (results identical) and batch rate vs CTAs per SM.
timeout 300 python tools/dbg_opts.py pack_tma 0,1,2 c2 c5 > gpurun_out/tma.log 2>&1
echo "rc=$?" >> gpurun_out/tma.log
