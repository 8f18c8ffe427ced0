set -x
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/sanitizer/r01_$tool.log 2>&1
  echo "$tool rc=$?"
done
