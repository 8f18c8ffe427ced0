# Same box A/B: the pre-packing attention kernel (BS_LIB=scripts/experiments/libbanaserve_prepack.so)
# vs the current one, decode-step flags, graph-timed, alternating.
mkdir -p gpurun_out/packab
for r in 1 2 3; do
  for lib in prepack current; do
    if [ $lib = prepack ]; then export BS_LIB=$PWD/scripts/experiments/libbanaserve_prepack.so; else unset BS_LIB; fi
    for c in C2_mha_B64_2048 C4_gqa8_mixed_B256 C3_gqa4_B8_8192 C3_gqa4_B1_8192; do
      timeout 120 python scripts/microbench.py --only attn --graph --step-flags --case $c 2>/dev/null | sed "s/^{/{\"lib\": \"$lib\", /"
    done
  done
done > gpurun_out/packab/mb.jsonl
