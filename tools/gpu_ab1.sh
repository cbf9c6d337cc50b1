set -u
mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/ab_batch.py pack_skip 0,1 c2 c4 c5 c3 > gpurun_out/ab_pack_skip.log 2>&1
timeout 600 python tools/ab_batch.py pack_tma 0,1,2 c2 c4 > gpurun_out/ab_pack_tma.log 2>&1
echo done
