# Experiment: programmatic dependent launch of the attention kernel (BS_ATTN_PDL=1: KV
# prefetch + block table before griddepcontrol.wait, q / outputs / workspace after).
# Parity of the whole GPU suite with PDL on, graph-timed microbench and the bench A/B.
mkdir -p gpurun_out/pdl
BS_ATTN_PDL=1 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pdl/pytest_pdl1.log 2>&1
echo "pytest pdl1 rc=$?"; tail -2 gpurun_out/pdl/pytest_pdl1.log
for round in 1 2 3; do
  for c in C3_gqa4_B1_8192 C3_gqa4_B8_8192 C3_gqa4_B32_8192 C2_mha_B64_2048 C4_gqa8_mixed_B256; do
    for pdl in 0 1; do
      BS_ATTN_PDL=$pdl timeout 120 python scripts/microbench.py --only attn --graph --case $c 2>/dev/null \
        | sed "s/^{/{\"pdl\": $pdl, /"
    done
  done
done > gpurun_out/pdl/microbench.jsonl
for pdl in 0 1 0 1; do
  BS_ATTN_PDL=$pdl timeout 900 python bench.py --no-cpu-baseline > gpurun_out/pdl/bench_pdl$pdl.$RANDOM.json 2>/dev/null
done
