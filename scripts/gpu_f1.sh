mkdir -p gpurun_out/f1
for r in 4 8; do for e in ce sm; do
  timeout 600 python scripts/bench_kvstore.py --requests $r --engine $e --json gpurun_out/f1/kvstore_${e}_r$r.json > /dev/null 2> gpurun_out/f1/kvstore_${e}_r$r.err
  echo "kvstore $e r$r rc=$?"
done; done
timeout 600 python -m pytest tests/test_gpu_kvstore.py -q > gpurun_out/f1/pytest_kvstore.log 2>&1; tail -1 gpurun_out/f1/pytest_kvstore.log
timeout 900 python scripts/bench_c5.py --json gpurun_out/f1/c5_share_n8.json > /dev/null 2> gpurun_out/f1/c5.err; echo "c5 rc=$?"
