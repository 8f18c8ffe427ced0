mkdir -p gpurun_out/exp6
for round in 1 2; do
  for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192 C3_gqa4_B32_8192 C2_mha_B64_2048 C4_gqa8_mixed_B256 C3_gqa4_B8_32768_1gpu; do
    timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null
  done
  for ns in 2 3 4; do for pdl in 0 1; do
    BS_ATTN_NSPLIT=$ns BS_ATTN_PDL=$pdl timeout 120 python scripts/microbench.py --only attn --graph --case C3_gqa4_B8_8192 2>/dev/null | sed "s/^{/{\"nsplit\": $ns, \"pdl\": $pdl, /"
  done; done
done > gpurun_out/exp6/microbench.jsonl
