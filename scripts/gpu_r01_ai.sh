set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 600 python scripts/microbench.py --only attn --graph --json gpurun_out/mb_graph.json > gpurun_out/mb_graph.log 2>&1
echo "graph rc=$?"
for cap in 4 8 16 32; do
  for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192; do
    BS_ATTN_MAX_BPS=$cap timeout 300 python scripts/microbench.py --only attn --graph --case $c > gpurun_out/mb_cap${cap}_$c.log 2>&1
  done
done
echo "caps done"
