set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 600 python scripts/bench_kvstore.py --json gpurun_out/kvstore_r4.json > gpurun_out/kvstore.log 2>&1
timeout 600 python scripts/bench_kvstore.py --requests 8 --json gpurun_out/kvstore_r8.json >> gpurun_out/kvstore.log 2>&1
echo "kvstore rc=$?"
