mkdir -p gpurun_out/f1b
timeout 600 python -m pytest tests/test_gpu_kvstore.py -q > gpurun_out/f1b/pytest_kvstore.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/f1b/pytest_kvstore.log
for r in 4 8; do for e in staged ce sm; do
  timeout 600 python scripts/bench_kvstore.py --requests $r --engine $e --json gpurun_out/f1b/kvstore_${e}_r$r.json > /dev/null 2> gpurun_out/f1b/kvstore_${e}_r$r.err
  echo "kvstore $e r$r rc=$?"
done; done
