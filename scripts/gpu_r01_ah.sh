set -x
mkdir -p gpurun_out
timeout 600 python scripts/microbench.py --only attn --graph --json gpurun_out/mb_graph.json > gpurun_out/mb_graph.log 2>&1
echo "graph rc=$?"
timeout 600 python scripts/microbench.py --only ragged --json gpurun_out/mb_ragged.json > gpurun_out/mb_ragged.log 2>&1
echo "ragged rc=$?"
timeout 600 python -m pytest tests/test_gpu_ragged.py -q > gpurun_out/pytest_ragged.log 2>&1
echo "pytest ragged rc=$?"
