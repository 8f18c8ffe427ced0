mkdir -p gpurun_out/deep2
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/deep2/pytest_gpu.log 2>&1
echo "gpu suite rc=$?"; tail -2 gpurun_out/deep2/pytest_gpu.log
for round in 1 2 3; do
  for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192 C2_mha_B64_2048 C4_gqa8_mixed_B256 C3_gqa4_B32_8192; do
    for pdl in 0 1; do
      BS_ATTN_PDL=$pdl timeout 120 python scripts/microbench.py --only attn --graph --case $c 2>/dev/null \
        | sed "s/^{/{\"pdl\": $pdl, /"
    done
  done
done > gpurun_out/deep2/microbench.jsonl
timeout 900 python bench.py > gpurun_out/deep2/bench.json 2> gpurun_out/deep2/bench.err
echo "bench rc=$?"
