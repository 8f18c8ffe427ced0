# Cluster merge (cap 8) tests + PDL pair timelines (eager and graph-captured pairs).
mkdir -p gpurun_out/cluster2
timeout 400 python -m pytest tests/test_gpu_cluster.py -q -x > gpurun_out/cluster2/pytest_cluster.log 2>&1
echo "cluster tests rc=$?"; tail -2 gpurun_out/cluster2/pytest_cluster.log
for pdl in 0 1; do
  BS_TIMELINE=1 BS_ATTN_PDL=$pdl timeout 300 python scripts/attn_timeline.py --pdl-pair --case C3_gqa4_B1_8192 \
    --case C3_gqa4_B8_8192 > gpurun_out/cluster2/pdl_pair_$pdl.jsonl 2> gpurun_out/cluster2/pdl_pair_$pdl.err
  echo "pdl pair $pdl rc=$?"
done
