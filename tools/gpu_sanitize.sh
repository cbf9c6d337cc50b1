# compute-sanitizer runs of tools/sanitize_run.py (every entry point on small
# masks), plus a positive control (tools/microbench/oob_probe: one OOB write
# memcheck must flag) so a clean log is known to come from an instrumented run.
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
$CS --tool memcheck --error-exitcode 9 tools/microbench/oob_probe > gpurun_out/sanitize_control.log 2>&1
echo "rc=$? (expected 9: the control's OOB write must be reported)" >> gpurun_out/sanitize_control.log
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  mode=""; [ $tool = racecheck ] && mode=quick
  t0=$(date +%s)
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 --target-processes all \
     python tools/sanitize_run.py $mode > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$? wall_s=$(( $(date +%s) - t0 ))" >> gpurun_out/sanitize_$tool.log
done
echo done
