set -u
mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 600 python tools/dbg_shard2.py > gpurun_out/dbg_shard2.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
