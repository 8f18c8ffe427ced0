mkdir -p gpurun_out/san2
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_cluster.py > gpurun_out/san2/$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san2/$tool.log
done
