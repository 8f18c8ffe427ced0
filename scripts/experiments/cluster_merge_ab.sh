# Cluster-merge check: the new tests, the attention / parity suites, then the graph-timed
# microbench A/B (BS_ATTN_CLUSTER=0 vs default) on the C3 / C2 / C4 shapes.
mkdir -p gpurun_out/cluster
timeout 240 python -m pytest tests/test_gpu_cluster.py -q -x > gpurun_out/cluster/pytest_cluster.log 2>&1
echo "cluster tests rc=$?"; tail -3 gpurun_out/cluster/pytest_cluster.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/cluster/pytest_gpu.log 2>&1
echo "gpu suite rc=$?"; tail -2 gpurun_out/cluster/pytest_gpu.log
for round in 1 2 3; do
  for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192 C3_gqa4_B32_8192 C2_mha_B64_2048 C4_gqa8_mixed_B256; do
    for cl in 0 1; do
      BS_ATTN_CLUSTER=$cl timeout 120 python scripts/microbench.py --only attn --graph --case $c 2>/dev/null \
        | sed "s/^{/{\"cluster\": $cl, /"
    done
  done
done > gpurun_out/cluster/microbench.jsonl
BS_TIMELINE=1 timeout 300 python scripts/attn_timeline.py --case C3_gqa4_B1_8192 --case C3_gqa4_B8_8192 \
  --json gpurun_out/cluster/timeline_c3.json > gpurun_out/cluster/timeline.log 2>&1
echo "timeline rc=$?"
