set -u
mkdir -p gpurun_out
make -s -C oracle >/dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 4 --warmup 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo done
