set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  mode=""; [ $tool = racecheck ] && mode=quick
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 --target-processes all \
     python tools/sanitize_run.py $mode > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
echo done
