# PDL with the late trigger for single-wave grids: tests, graph-timed microbench A/B,
# PDL pair timelines.
mkdir -p gpurun_out/pdl2
timeout 600 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_pdl.py -q -x > gpurun_out/pdl2/pytest.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/pdl2/pytest.log
BS_ATTN_PDL=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster.py -q -x > gpurun_out/pdl2/pytest_pdl1.log 2>&1
echo "tests pdl1 rc=$?"; tail -2 gpurun_out/pdl2/pytest_pdl1.log
for round in 1 2 3; do
  for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192 C3_gqa4_B32_8192 C2_mha_B64_2048 C4_gqa8_mixed_B256; do
    for pdl in 0 1; do
      BS_ATTN_PDL=$pdl timeout 120 python scripts/microbench.py --only attn --graph --case $c 2>/dev/null \
        | sed "s/^{/{\"pdl\": $pdl, /"
    done
  done
done > gpurun_out/pdl2/microbench.jsonl
for pdl in 0 1; do
  BS_TIMELINE=1 BS_ATTN_PDL=$pdl timeout 300 python scripts/attn_timeline.py --pdl-pair --case C3_gqa4_B1_8192 \
    --case C3_gqa4_B8_8192 > gpurun_out/pdl2/pdl_pair_$pdl.jsonl 2> gpurun_out/pdl2/pdl_pair_$pdl.err
  echo "pdl pair $pdl rc=$?"
done
