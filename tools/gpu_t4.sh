set -u
mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/raw_e2e.py 32 > gpurun_out/raw_e2e.json 2> gpurun_out/raw_e2e.err
echo done
