# Flag merge: targeted tests first (short timeout), full suite, A/B microbench, timeline.
mkdir -p gpurun_out/fm
timeout 300 python -m pytest tests/test_gpu_cluster.py -q -x > gpurun_out/fm/pytest_cluster.log 2>&1
echo "cluster tests rc=$?"; tail -2 gpurun_out/fm/pytest_cluster.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/fm/pytest_gpu.log 2>&1
echo "gpu suite rc=$?"; tail -2 gpurun_out/fm/pytest_gpu.log
for round in 1 2 3; do
  for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192; do
    for fm in 0 1; do
      BS_ATTN_FLAGMERGE=$fm timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null | sed "s/^{/{\"fm\": $fm, /"
      BS_ATTN_FLAGMERGE=$fm BS_ATTN_CLUSTER=0 timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null | sed "s/^{/{\"fm\": $fm, \"nocluster\": 1, /"
    done
  done
done > gpurun_out/fm/microbench.jsonl
BS_TIMELINE=1 BS_ATTN_PDL=1 timeout 300 python scripts/attn_timeline.py --pdl-pair --case C3_gqa4_B1_8192 > gpurun_out/fm/pdl_pair.jsonl 2> gpurun_out/fm/pdl_pair.err
BS_TIMELINE=1 timeout 300 python scripts/attn_timeline.py --case C3_gqa4_B1_8192 --case C3_gqa4_B8_8192 --json gpurun_out/fm/timeline.json > /dev/null 2>&1
echo done
