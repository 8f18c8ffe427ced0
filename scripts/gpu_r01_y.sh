set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "graph or bench_step" > gpurun_out/pytest_graph.log 2>&1
echo "pytest rc=$?"
for c in 0 128 64 32; do
BS_ATTN_MAX_BPS=$c timeout 600 python scripts/microbench.py --only attn --json gpurun_out/micro_bps$c.json > gpurun_out/micro_bps$c.log 2>&1
done
echo "micro rc=$?"
