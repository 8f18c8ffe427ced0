set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
for e in ce sm; do for r in 4 8; do
timeout 600 python scripts/bench_kvstore.py --engine $e --requests $r --json gpurun_out/kvstore_${e}_r${r}.json >> gpurun_out/kvstore.log 2>&1
done; done
echo "kvstore rc=$?"
