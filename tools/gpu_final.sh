#!/bin/bash
# Round-end evidence: parity tests, smoke, default bench (C4 headline + C2,
# CPU baseline), per-workload bench lines, reference arm, batch trace, ncu
# launch lists + full captures, sanitizers.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python tools/stress_parity.py 600 21000 > $OUT/stress_parity.txt 2>&1; echo "rc=$?" >> $OUT/stress_parity.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
for w in c1 c3 c5; do
  timeout 600 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu-baseline > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
timeout 600 python bench.py --steps 5 --warmup 3 --workload c3 --split > $OUT/bench_c3_split.json 2> $OUT/bench_c3_split.err
timeout 600 python bench.py --split --workload c3 --sim-shards 2 4 8 --steps 7 --warmup 3 > $OUT/bench_c3_slab_sim.json 2> $OUT/bench_c3_slab_sim.err
timeout 300 python bench.py --split --workload c2 --sim-shards 2 4 --steps 7 --warmup 3 > $OUT/bench_c2_slab_sim.json 2> $OUT/bench_c2_slab_sim.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
SC_TRACE=1 timeout 300 python tools/batch_probe.py c4 300 - > $OUT/trace_c4.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c2.csv python tools/one_roi.py c2 > $OUT/ncu_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c3.csv python tools/one_roi.py c3 > $OUT/ncu_bench_c3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c4.csv python tools/one_roi.py c4 tma > $OUT/ncu_bench_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c3_slab.csv python tools/shard_roi.py c3 2 slab > $OUT/ncu_bench_slab.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"pack_bits|mc_cells|scan_all|scatter_all|boxes_extremes|unit_filter|plane_boxes|plane_lb|plane_filter|diam_pass1|diam_refine" -s 12 -c 12 \
    -o $OUT/prof -f python tools/one_roi.py c2 > $OUT/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pack_bits_tma" -s 0 -c 1 \
    -o $OUT/prof_tma -f python tools/one_roi.py c4 tma > $OUT/ncu_tma.log 2>&1
# (compute-sanitizer runs: tools/gpu_sanitize.sh -- closed on the GPU pool since late round 2)
echo done
